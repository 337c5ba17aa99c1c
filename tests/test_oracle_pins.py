"""Pins for the CPU oracle (oracle/) against what the paper and the
mathematics fix — never against the oracle itself.

* paper listing verdicts (tests/golden/listings.txt, each line cited);
* the C1 tree-reduction closed form (derived below from the race definition);
* classical vector clocks over EVERY barrier-respecting interleaving
  (SPEC.md:416-424, 612): the static set must equal the dynamic one on each;
* pairwise == bucketed modes on random programs;
* the two-thread property;
* schedule counts; clock overflow;
* the scope lemma (racy + >=2 blocks <=> a cross-block racing pair).
"""
import os
import random

import pytest

import oracle
from oracle import vclock
from tracegen import format as tf
from tracegen import programs as tp

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "listings.txt")


def _golden():
    rows = []
    for line in open(GOLDEN):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        head, words, scope, cite = [x.strip() for x in line.split("|")]
        name, b, w, l, p = head.split()
        exp = [] if words == "-" else [int(x) for x in words.split(",")]
        rows.append((name, int(b), int(w), int(l), int(p), exp, scope, cite))
    return rows


def _make(name, b, w, l, p):
    if name == "listing1":
        return tp.listing1(b, w, l)
    if name == "listing2":
        return tp.listing2(b, w, l)
    return tp.listing4(b, w, l, p)


@pytest.mark.parametrize("row", _golden(), ids=lambda r: f"{r[0]}-{r[1]}x{r[2]}x{r[3]}")
@pytest.mark.parametrize("mode", [oracle.PAIRWISE, oracle.BUCKETED])
def test_paper_listings(row, mode):
    name, b, w, l, p, exp, scope, cite = row
    res = oracle.check(_make(name, b, w, l, p), mode=mode)
    assert [r.word for r in res.races] == exp, cite
    if exp:
        want = oracle.SCOPE_GRID if scope == "GRID" else oracle.SCOPE_BLOCK
        assert all(r.scope == want for r in res.races), cite
    assert res.flags == 0


def test_listing2_all_block_counts():
    # ">= 2 blocks" racy on data[0..T-2]; 1 block race-free
    for blocks in (1, 2, 3):
        for (w, l) in ((1, 2), (2, 2), (1, 5), (3, 3)):
            t = w * l
            res = oracle.check(tp.listing2(blocks, w, l))
            exp = [] if blocks == 1 else list(range(t - 1))
            assert [r.word for r in res.races] == exp


def test_c1_closed_form():
    """C1: barrier after reduction step s removed merges step s
    (writes s[i], i<s, lane i%32) with step s/2 (reads s[i], s[i+s/2],
    i<s/2, lane i%32).  s[j], j in [s/2, s), is written by lane j%32 and read
    by lane (j-s/2)%32 with no barrier between: distinct lanes (a race) iff
    s/2 is not a multiple of 32, i.e. s <= 32.  Hence racy = [s/2, s) for
    s in {32,16,8,4,2}, empty otherwise.  All in one block -> BLOCK scope."""
    for removed in (None, "load", 128, 64, 32, 16, 8, 4, 2, 1):
        tr = tp.c1_tree_reduction(removed=removed)
        res = oracle.check(tr, mode=oracle.BUCKETED)
        if removed in (32, 16, 8, 4, 2):
            exp = list(range(removed // 2, removed))
        else:
            exp = []
        assert [r.word for r in res.races] == exp, removed
        assert all(r.space == tf.SPACE_SHARED and r.block == 0 and r.scope == oracle.SCOPE_BLOCK
                   for r in res.races)
        # 10,232 checked accesses per launch (8 x (512 + 765 + 2))
        assert res.n_accesses == 10232


def test_c1_pairwise_equals_bucketed():
    tr = tp.c1_tree_reduction(removed=16, rounds=2)
    assert oracle.check(tr, mode=oracle.PAIRWISE) == oracle.check(tr, mode=oracle.BUCKETED)


def _static_as_dict(res):
    return {(r.space, r.block, r.word): r.scope for r in res.races}


def test_vclock_every_interleaving_equals_static():
    """on every interleaving the vector-clock verdict equals
    the static happens-before set (all events execute in each complete run)."""
    rng = random.Random(1234)
    n_sched = 0
    for _ in range(150):
        tr = tp.random_program(rng, max_blocks=2, max_warps=2, max_lanes=2, max_slots=3,
                               n_words=2, spaces=(0, 1))
        th = vclock.thread_events(tr)[0]
        static = _static_as_dict(oracle.check(tr, mode=oracle.PAIRWISE))
        for sched in vclock.enumerate_schedules(th, cap=300):
            assert vclock.vclock_races(th, sched) == static
            n_sched += 1
    assert n_sched > 5000


def test_race_classes_listings():
    """Classes follow from the listings' kinds (bit0 W-W, bit1 R-W, bit2 A-W, bit3 A-R):
    Listing 1: every thread reads then writes data[0] -> R-W and W-W.
    Listing 2 at 2 blocks: data[0] read by all, written by thread 1 of
    each block -> R-W and W-W; data[k>0] only written (by thread k+1 of each
    block) -> W-W.  Listing 4: data[j] read by threads j, j-1 and
    written by thread j-1 only -> R-W."""
    assert oracle.check(tp.listing1(1, 1, 4)).classes == [3]
    r = oracle.check(tp.listing2(2, 1, 4))
    assert [x.word for x in r.races] == [0, 1, 2] and r.classes == [3, 1, 1]
    assert set(oracle.check(tp.listing4(1, 1, 8, 8)).classes) == {2}
    two = lambda k1, k2: tp.from_thread_events(1, 1, 2, {(0, 0, 0): [k1(0)], (0, 0, 1): [k2(0)]})  # noqa: E731
    assert oracle.check(two(tf.A, tf.W)).classes == [4]
    assert oracle.check(two(tf.R, tf.A)).classes == [8]


def test_vclock_classes_every_interleaving():
    """The static classes equal the classes of the racing pairs a vector-clock
    detector sees along every interleaving."""
    rng = random.Random(4321)
    n = 0
    for _ in range(120):
        tr = tp.random_program(rng, max_blocks=2, max_warps=2, max_lanes=2, max_slots=3, n_words=2,
                               spaces=(0, 1))
        th = vclock.thread_events(tr)[0]
        res = oracle.check(tr, mode=oracle.PAIRWISE)
        static = {(r.space, r.block, r.word): c for r, c in zip(res.races, res.classes)}
        for sched in vclock.enumerate_schedules(th, cap=200):
            assert vclock.vclock_race_classes(th, sched) == static
            n += 1
    assert n > 3000


def test_pairwise_equals_bucketed_random():
    rng = random.Random(99)
    for i in range(400):
        tr = tp.random_program(rng, max_blocks=3, max_warps=3, max_lanes=4, max_slots=6,
                               n_words=3, spaces=(0, 1), n_kernels=rng.randint(1, 2))
        a = oracle.check(tr, mode=oracle.PAIRWISE)
        b = oracle.check(tr, mode=oracle.BUCKETED)
        assert a == b, i


def test_two_thread_property():
    """under barrier-only, data-independent control a race is
    discoverable within two threads."""
    rng = random.Random(7)
    checked = 0
    for _ in range(300):
        tr = tp.random_program(rng, max_blocks=2, max_warps=2, max_lanes=2, max_slots=3, n_words=2)
        th = vclock.thread_events(tr)[0]
        static = _static_as_dict(oracle.check(tr))
        if not static:
            continue
        found = {}
        for pair in vclock.thread_pairs(th):
            sub = vclock.project(th, set(pair))
            sched = next(vclock.enumerate_schedules(sub))
            for a, s in vclock.vclock_races(sub, sched).items():
                found[a] = max(found.get(a, 0), s)
        assert found == static
        checked += 1
    assert checked > 50


def test_schedule_counts():
    # 2 threads x 1 event -> 2 schedules; 2 x 2 events -> C(4,2) = 6
    tr = tp.from_thread_events(1, 1, 2, {(0, 0, 0): [tf.R(0)], (0, 0, 1): [tf.R(1)]})
    assert len(list(vclock.enumerate_schedules(vclock.thread_events(tr)[0]))) == 2
    tr = tp.from_thread_events(1, 1, 2, {(0, 0, 0): [tf.R(0), tf.R(1)], (0, 0, 1): [tf.R(2), tf.R(3)]})
    assert len(list(vclock.enumerate_schedules(vclock.thread_events(tr)[0]))) == 6
    # Listing 2 on 1x1x2: both reads precede every post-barrier event
    th = vclock.thread_events(tp.listing2(1, 1, 2))[0]
    n = 0
    for sched in vclock.enumerate_schedules(th):
        run = vclock._Run(th)
        kinds = [run.exec(t)[0] for t in sched]
        accs = [e for e in kinds if e[0] == "acc"]
        assert [e[3] for e in accs] == [tf.OP_READ, tf.OP_READ, tf.OP_WRITE]
        n += 1
    assert n > 1


def test_clock_overflow():
    """detection discontinued with a warning after reporting any
    previously identified races.  SPEC.md:617: bc_bits = 2 and 4 barriers."""
    ev = {(0, 0, 0): [tf.W(0), tf.SYNCTHREADS, tf.SYNCTHREADS, tf.SYNCTHREADS, tf.SYNCTHREADS, tf.W(1)],
          (0, 0, 1): [tf.W(0), tf.SYNCTHREADS, tf.SYNCTHREADS, tf.SYNCTHREADS, tf.SYNCTHREADS, tf.W(1)]}
    tr = tp.from_thread_events(1, 1, 2, ev)
    full = oracle.check(tr)
    assert [r.word for r in full.races] == [0, 1] and full.flags == 0
    over = oracle.check(tr, bc_bits=2)
    assert [r.word for r in over.races] == [0]            # race before the overflow kept
    assert over.flags & oracle.F_CLOCK_OVERFLOW
    three = tp.from_thread_events(1, 1, 2, {k: v[:4] + v[5:] for k, v in ev.items()})
    assert oracle.check(three, bc_bits=2).flags == 0      # 3 barriers fit in 2 bits


def test_kernel_boundary_orders():
    k1 = tf.build_kernel(1, 1, 2, lambda b, w, l: [tf.W(0)] if l == 0 else [])
    k2 = tf.build_kernel(1, 1, 2, lambda b, w, l: [tf.R(0)] if l == 1 else [])
    assert oracle.check(tf.make_trace([k1, k2])).races == []
    k3 = tf.build_kernel(1, 1, 2, lambda b, w, l: [tf.W(0)])
    res = oracle.check(tf.make_trace([k1, k3]))
    assert [(r.kernel, r.word) for r in res.races] == [(1, 0)]


def test_atomics_reading():
    """Reading R1: A-A never races; A-R and A-W do."""
    def two(k1, k2):
        return tp.from_thread_events(1, 1, 2, {(0, 0, 0): [k1(0)], (0, 0, 1): [k2(0)]})
    assert oracle.check(two(tf.A, tf.A)).races == []
    assert len(oracle.check(two(tf.A, tf.R)).races) == 1
    assert len(oracle.check(two(tf.W, tf.A)).races) == 1
    assert oracle.check(two(tf.R, tf.R)).races == []


def test_shared_instances_are_per_block():
    tr = tp.from_thread_events(2, 1, 1, {(0, 0, 0): [tf.W(5, tf.SPACE_SHARED)],
                                         (1, 0, 0): [tf.W(5, tf.SPACE_SHARED)]}, smem_words=8)
    assert oracle.check(tr).races == []
    tr = tp.from_thread_events(2, 1, 1, {(0, 0, 0): [tf.W(5)], (1, 0, 0): [tf.W(5)]})
    assert [(r.word, r.scope) for r in oracle.check(tr).races] == [(5, oracle.SCOPE_GRID)]


def test_scope_lemma():
    """For a racy address: a cross-block racing pair exists iff >= 2 blocks
    accessed it (SURVEY §8(c) Output 2) — brute force on random programs."""
    from tests.helpers import accesses_by_address
    rng = random.Random(5)
    for _ in range(300):
        tr = tp.random_program(rng, max_blocks=3, max_warps=2, max_lanes=2, max_slots=5, n_words=2)
        res = oracle.check(tr, mode=oracle.PAIRWISE)
        acc = accesses_by_address(tr)
        for r in res.races:
            blocks = {a[0][0] for a in acc[(r.kernel, r.space, r.block, r.word)]}
            assert (r.scope == oracle.SCOPE_GRID) == (len(blocks) >= 2)


def test_barrier_divergence_flag():
    # lane 0 syncs, lane 1 does not: built by hand (the builder refuses it)
    import numpy as np
    rows = np.full((1, 2, 32), tf.NOP, dtype=np.uint64)
    rows[0, 0, 0] = tf.SYNCTHREADS
    rows[0, 1, 1] = tf.W(0)
    tr = tf.make_trace([tf.kernel_from_rows(1, 1, 2, rows)])
    assert oracle.check(tr).flags & oracle.F_BARRIER_DIVERGENCE
    with pytest.raises(tf.BarrierDivergence):
        tp.from_thread_events(1, 1, 2, {(0, 0, 0): [tf.SYNCTHREADS], (0, 0, 1): [tf.W(0)]})


def test_undefined_control_code_is_no_barrier():
    """The oracle's model-violation branch (reading R12 in DESIGN.md): the trace
    format defines control words 0 NOP, 1 __syncthreads, 2 __syncwarp; any
    other code is flagged and is NOT a barrier.  Pinned by the barrier
    semantics (§II-B): lane 0 writes word 0, then every lane
    holds the code, then lane 1 reads word 0.  Had the code been a __syncwarp
    the two accesses would be ordered (same warp, later warp epoch) and there
    would be no race; as no barrier they are unordered and word 0 races,
    BLOCK scope (one block)."""
    import numpy as np
    for code in (3, 7, 12345):
        rows = np.full((1, 3, 32), tf.NOP, dtype=np.uint64)
        rows[0, 0, 0] = tf.W(0)
        rows[0, 1, :] = tf.encode(tf.OP_CTRL, 0, code)
        rows[0, 2, 1] = tf.R(0)
        tr = tf.make_trace([tf.kernel_from_rows(1, 1, 2, rows)])
        for mode in (oracle.PAIRWISE, oracle.BUCKETED):
            res = oracle.check(tr, mode=mode)
            assert res.flags == oracle.F_MODEL_VIOLATION
            assert [(r.word, r.scope) for r in res.races] == [(0, oracle.SCOPE_BLOCK)]
        rows[0, 1, :] = tf.SYNCWARP
        res = oracle.check(tf.make_trace([tf.kernel_from_rows(1, 1, 2, rows)]))
        assert res.races == [] and res.flags == 0
        # an undefined code orders nothing: the set equals that of the same trace with a NOP there
        rows[0, 1, :] = tf.NOP
        assert [r.word for r in oracle.check(tf.make_trace([tf.kernel_from_rows(1, 1, 2, rows)])).races] == [0]


def _masked_syncwarp_trace(barrier=tf.SYNCWARP, lanes_in=(0, 1)):
    """1 block, 1 warp, 3 active lanes.  The lanes `lanes_in` hold a __syncwarp
    record on row 2 (lanes (0, 1): a __syncwarp(0b011) in CUDA terms).  Lane 0
    writes words 1 and 0 before it; after it lane 1 reads word 0 and lane 2
    reads word 1."""
    import numpy as np
    rows = np.full((1, 4, 32), tf.NOP, dtype=np.uint64)
    rows[0, 0, 0] = tf.W(1)
    rows[0, 1, 0] = tf.W(0)
    for l in lanes_in:
        rows[0, 2, l] = barrier
    rows[0, 3, 1] = tf.R(0)
    rows[0, 3, 2] = tf.R(1)
    return tf.make_trace([tf.kernel_from_rows(1, 1, 3, rows)])


def test_masked_syncwarp_conservative_reading():
    """Reading R8: a __syncwarp that only some lanes hold is
    __syncwarp(mask) with a sub-warp mask ("takes a mask
    argument"); a scalar warp clock cannot express it, so the oracle flags a
    model violation and adds no happens-before edge.  Pins:
      * exact semantics (vector clocks where the barrier joins exactly the
        masked lanes, over every interleaving): word 0 is ordered (lanes 0
        and 1 are both in the mask), word 1 races (lane 2 is not);
      * the oracle's set is a superset of the exact one (sound), and equals
        the set of the same trace with the masked barrier removed;
      * a full-warp __syncwarp in the same place orders both."""
    tr = _masked_syncwarp_trace()
    th = vclock.thread_events(tr)[0]
    exact = set()
    n = 0
    for sched in vclock.enumerate_schedules(th):
        exact |= set(vclock.vclock_races(th, sched))
        n += 1
    assert n > 1 and exact == {(0, 0xFFFFFFFF, 1)}
    for mode in (oracle.PAIRWISE, oracle.BUCKETED):
        res = oracle.check(tr, mode=mode)
        assert res.flags == oracle.F_MODEL_VIOLATION
        got = {(r.space, r.block, r.word) for r in res.races}
        assert got >= exact and got == {(0, 0xFFFFFFFF, 0), (0, 0xFFFFFFFF, 1)}
    nop = _masked_syncwarp_trace(barrier=tf.NOP)
    assert [tuple(r) for r in oracle.check(nop).races] == [tuple(r) for r in oracle.check(tr).races]
    full = oracle.check(_masked_syncwarp_trace(lanes_in=(0, 1, 2)))
    assert full.races == [] and full.flags == 0


def _tile_example(declared: bool):
    """T = 2 lanes per tile (tiles {0,1}, {2,3}).  Lane 0 writes word 0 and
    lane 2 word 1; tile 0 then meets a tile barrier (lanes 0 and 1 hold the
    __syncwarp record), tile 1 does not; then lane 1 reads word 0 and lane 3
    reads word 1."""
    import numpy as np
    rows = np.full((1, 3, 32), tf.NOP, dtype=np.uint64)
    rows[0, 0, 0] = tf.W(0)
    rows[0, 0, 2] = tf.W(1)
    rows[0, 1, 0] = tf.SYNCWARP
    rows[0, 1, 1] = tf.SYNCWARP
    rows[0, 2, 1] = tf.R(0)
    rows[0, 2, 3] = tf.R(1)
    k = tf.kernel_from_rows(1, 1, 4, rows)
    k.tile_log2 = 1 if declared else 0
    return tf.make_trace([k])


def test_tile_barriers_exact():
    """Warp tiles (PAPER.md:264 __syncwarp's mask; the paper's future work,
    PAPER.md:1054): a kernel that declares T-lane tiles treats an aligned
    partial __syncwarp row as one barrier per tile, exactly (reading R8).
    Pinned by hand (word 0 is ordered by tile 0's barrier, word 1 is not:
    tile 1 never synchronised) and by vector clocks whose tile barriers join
    exactly the tile's lanes over every interleaving; undeclared, the same row
    is a sub-warp mask handled conservatively (both words, model violation)."""
    tr = _tile_example(True)
    th = vclock.thread_events(tr)[0]
    exact = set()
    for sched in vclock.enumerate_schedules(th):
        exact |= set(vclock.vclock_races(th, sched))
    assert exact == {(0, 0xFFFFFFFF, 1)}
    for mode in (oracle.PAIRWISE, oracle.BUCKETED):
        res = oracle.check(tr, mode=mode)
        assert res.flags == 0
        assert {(r.space, r.block, r.word) for r in res.races} == exact
    und = oracle.check(_tile_example(False))
    assert und.flags == oracle.F_MODEL_VIOLATION and [r.word for r in und.races] == [0, 1]


@pytest.mark.slow
def test_tile_programs_vector_clocks_and_modes():
    """Random tile programs (tiny: every interleaving enumerated) — the
    oracle's static set equals the vector-clock set on every interleaving;
    larger ones — pairwise == bucketed."""
    rng = random.Random(91)
    n_checked = 0
    for _ in range(60):
        tr = tp.random_tile_program(rng, blocks=rng.randint(1, 2), warps=1, lanes=4, tile_log2=rng.choice([1, 2]),
                                    slots=rng.randint(2, 4), n_words=2, p_tile=0.35, p_sync=0.1)
        th = vclock.thread_events(tr)[0]
        want = {(r.space, r.block, r.word) for r in oracle.check(tr, mode=oracle.PAIRWISE).races}
        for i, sched in enumerate(vclock.enumerate_schedules(th, cap=400)):
            assert set(vclock.vclock_races(th, sched)) == want
            n_checked += 1
    assert n_checked > 1000
    for _ in range(30):
        tr = tp.random_tile_program(rng, blocks=3, warps=2, lanes=32, tile_log2=rng.choice([1, 2, 3, 4]), slots=14,
                                    n_words=20, spaces=(0, 1))
        a = oracle.check(tr, mode=oracle.PAIRWISE)
        b = oracle.check(tr, mode=oracle.BUCKETED)
        assert [tuple(r) for r in a.races] == [tuple(r) for r in b.races] and a.flags == b.flags == 0
