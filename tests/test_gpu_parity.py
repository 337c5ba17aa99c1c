"""GPU parity: the CUDA path through the C ABI vs the CPU oracle, element by
element (racy address + scope), bit-exact — integer work (north_star).

Covers: paper listings, C1 all variants, random programs over grids up to
32 warps x 32 lanes with shared/global/atomics/both barriers and multiple
kernels, schedule fuzzing (coalescing off, lane and block permutations),
ring overflow fallback, clock overflow, shard emulation, host-buffer replay.
"""
import random

import numpy as np
import pytest

import oracle
from tracegen import format as tf
from tracegen import programs as tp

pytestmark = pytest.mark.gpu


def hr():
    from paper_2401_04701_b200 import hirace
    return hirace


def gpu_set(trace, **kw):
    races, flags = hr().check_trace(trace, **kw)
    return [tuple(r) for r in races], flags


def oracle_set(trace, **kw):
    res = oracle.check(trace, **kw)
    return [tuple(r) for r in res.races], res.flags


def test_listings():
    for tr in (tp.listing1(1, 1, 2), tp.listing1(2, 2, 2), tp.listing1(64, 8, 32), tp.listing2(1, 1, 4),
               tp.listing2(2, 2, 2), tp.listing2(1, 32, 32), tp.listing2(3, 4, 32), tp.listing4(1, 1, 4, 4),
               tp.listing4(1, 4, 32, 100), tp.listing4(2, 1, 2, 4)):
        assert gpu_set(tr) == oracle_set(tr)


@pytest.mark.parametrize("removed", [None, "load", 128, 64, 32, 16, 8, 4, 2, 1])
def test_c1_tree_reduction(removed):
    tr = tp.c1_tree_reduction(removed=removed)
    g, fl = gpu_set(tr)
    o, ofl = oracle_set(tr)
    assert g == o and fl == ofl == 0


def _random_batch(seed, n, **kw):
    rng = random.Random(seed)
    kernels = []
    for _ in range(n):
        t = tp.random_program(rng, **kw)
        blocks, warps, lanes, smem, _ = (int(x) for x in t.kdesc[0, :5])
        rows = [t.rec[int(t.warp_off[w]) * 32: int(t.warp_off[w + 1]) * 32].reshape(-1, 32)
                for w in range(blocks * warps)]
        k = tf.Kernel(blocks, warps, lanes, smem)
        k.rows = rows
        kernels.append(k)
    return tf.make_trace(kernels)


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("options", [16, 32, 256, 512])
def test_random_small_family(seed, options):
    tr = _random_batch(seed, 300, max_blocks=2, max_warps=2, max_lanes=2, max_slots=5, n_words=2,
                       spaces=(0, 1))
    assert gpu_set(tr, options=options) == oracle_set(tr)


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("options", [16, 32, 256, 512, 65536])
def test_random_wide_grids(seed, options):
    """Full warps and many warps: exercises MATCH coalescing, multi-lane folds,
    CAS contention, several tiles of the shadow and ragged warp lengths, in
    both the row and the pooled replay."""
    tr = _random_batch(100 + seed, 40, max_blocks=6, max_warps=8, max_lanes=32, max_slots=12,
                       n_words=40, spaces=(0, 1), p_barrier=0.25, p_skip=0.5)
    g, fl = gpu_set(tr, options=options)
    o, ofl = oracle_set(tr)
    assert g == o and fl == ofl
    assert len(o) > 10


@pytest.mark.parametrize("options", [16, 32, 256, 512, 65536])
def test_hot_words_contention(options):
    """Few words, 32 warps x 32 lanes x 16 blocks: heavy CAS retry storms."""
    tr = _random_batch(7, 10, max_blocks=16, max_warps=32, max_lanes=32, max_slots=8, n_words=3,
                       spaces=(0, 1), p_skip=0.2)
    assert gpu_set(tr, options=options) == oracle_set(tr)
    tr = _random_batch(8, 10, max_blocks=16, max_warps=32, max_lanes=32, max_slots=8, n_words=3,
                       kinds="RA", spaces=(0, 1), p_skip=0.2)
    assert gpu_set(tr, options=options) == oracle_set(tr)


@pytest.mark.parametrize("options", [1, 2, 3, 8, 2048, 16, 32, 32 | 1, 32 | 2048, 64, 64 | 32, 256, 256 | 1,
                                     256 | 2048, 512, 512 | 1, 512 | 2, 512 | 2048, 256 | 1024,
                                     256 | 1024 | 2048, 16 | 2048 | 64, 65536, 65536 | 1, 65536 | 2048,
                                     65536 | 8192])
def test_ablations_same_result(options):
    """Coalescing off / fast exits off / no speculation / forced row or pooled
    replay change the commit order and the traffic, never the result
    (schedule independence)."""
    tr = _random_batch(21, 60, max_blocks=4, max_warps=4, max_lanes=32, max_slots=10, n_words=8,
                       spaces=(0, 1))
    assert gpu_set(tr, options=options) == oracle_set(tr)


def test_lane_and_block_permutation_invariance():
    rng = random.Random(3)
    tr = _random_batch(31, 30, max_blocks=4, max_warps=2, max_lanes=32, max_slots=8, n_words=10,
                       spaces=(0,))
    base, _ = gpu_set(tr)
    perm = list(range(32))
    rng.shuffle(perm)
    rec = tr.rec.reshape(-1, 32)[:, perm].reshape(-1).copy()
    # lanes of a row are remapped: only words + scopes are compared (global space)
    tr2 = tf.Trace(rec, tr.kdesc.copy(), tr.warp_off.copy())
    for k in range(tr2.kdesc.shape[0]):
        tr2.kdesc[k, 2] = 32
    assert gpu_set(tr2) == oracle_set(tr2)
    assert oracle_set(tr2)[0] == base


def test_repeated_runs_identical():
    tr = _random_batch(41, 20, max_blocks=8, max_warps=8, max_lanes=32, max_slots=10, n_words=4,
                       spaces=(0, 1))
    o = oracle_set(tr)
    for _ in range(5):
        assert gpu_set(tr) == o


@pytest.mark.parametrize("options", [0, 64])
def test_reused_context_across_replays(options):
    """One ctx, several replays of multi-kernel traces: every kernel starts from
    a clean shadow (kernel boundary, a11), with one or two shadow buffers."""
    h = hr()
    trs = [_random_batch(70 + i, 12, max_blocks=4, max_warps=4, max_lanes=32, max_slots=10, n_words=64,
                         spaces=(0, 1)) for i in range(3)]
    ck = h.Checker(4096, 64, options=options)
    for tr in trs + trs[::-1]:
        ck.reset()
        ck.replay(h.DeviceTrace.from_trace(tr))
        races, fl, _ = ck.report()
        assert ([tuple(r) for r in races], fl) == oracle_set(tr)
    ck.close()


@pytest.mark.parametrize("options", [0, 64])
def test_ring_overflow_falls_back_to_shadow_scan(options):
    # one kernel, many racy global words
    tr = tp.listing2(4, 8, 32)
    g, fl = gpu_set(tr, ring_capacity=8, options=options)
    o, _ = oracle_set(tr)
    assert fl & hr().HR_F_RING_OVERFLOW
    assert g == o


def test_clock_overflow():
    ev = {(0, 0, 0): [tf.W(0)] + [tf.SYNCTHREADS] * 4 + [tf.W(1)],
          (0, 0, 1): [tf.W(0)] + [tf.SYNCTHREADS] * 4 + [tf.W(1)]}
    tr = tp.from_thread_events(1, 1, 2, ev)
    g, fl = gpu_set(tr, bc_bits=2, wc_bits=30)
    o, ofl = oracle_set(tr, bc_bits=2, wc_bits=30)
    assert g == o and fl == ofl == hr().HR_F_CLOCK_OVERFLOW
    assert [r[3] for r in g] == [0]


def test_shard_emulation_union_equals_single():
    """N address shards on one GPU, concatenated, equal the
    single-GPU result (words are independent FSMs)."""
    h = hr()
    tr = _random_batch(51, 20, max_blocks=4, max_warps=4, max_lanes=32, max_slots=10, n_words=3000,
                       spaces=(0, 1))
    gmax, smem = h.trace_extent(tr)
    full, _ = gpu_set(tr)
    for n, g in ((2, 9), (4, 9), (8, 9), (8, 5), (4, 6), (8, 0), (4, 3)):
        union = []
        for r in range(n):
            ck = h.Checker(gmax, smem, shard=(r, n), granule_log2=g)
            ck.replay(h.DeviceTrace.from_trace(tr))
            races, _, _ = ck.report()
            ck.close()
            union += [tuple(x) for x in races]
        assert sorted(union) == full


def test_shard_ring_overflow_scan():
    """A shard whose race ring overflows falls back to the shadow scan of its
    (single) kernel, which maps local granules back through the owner
    function's inverse (hr_shard_granule): the union over shards still equals
    the oracle's set."""
    h = hr()
    tr = tp.listing2(8, 8, 32)                       # one kernel, many racy global words
    gmax, smem = h.trace_extent(tr)
    full, _ = oracle_set(tr)
    assert len(full) > 64
    for n, g in ((4, 9), (8, 0), (2, 5), (4, 3)):
        union, ov = [], 0
        for r in range(n):
            ck = h.Checker(gmax, smem, shard=(r, n), granule_log2=g, ring_capacity=4)
            ck.replay(h.DeviceTrace.from_trace(tr))
            races, fl, _ = ck.report()
            ck.close()
            ov |= fl & h.HR_F_RING_OVERFLOW
            union += [tuple(x) for x in races]
        assert ov
        assert sorted(union) == full


def test_host_buffer_replay():
    h = hr()
    tr = tp.c1_tree_reduction(removed=8)
    gmax, smem = h.trace_extent(tr)
    ck = h.Checker(gmax, smem)
    ck.replay_host(tr)
    races, fl, _ = ck.report()
    assert [tuple(r) for r in races] == oracle_set(tr)[0]


def test_empty_and_degenerate():
    h = hr()
    # a kernel with no accesses at all
    tr = tf.single_kernel(2, 2, 32, lambda b, w, l: [tf.SYNCTHREADS])
    assert gpu_set(tr) == ([], 0)
    # single thread: never races
    tr = tp.from_thread_events(1, 1, 1, {(0, 0, 0): [tf.W(0), tf.R(0), tf.A(0), tf.W(0)]})
    assert gpu_set(tr) == ([], 0)


@pytest.mark.parametrize("options", [16, 32])
def test_compact_format_same_result(options):
    """HR_TRACE_C32 (u32 word + op/space byte per record) decodes to the same
    records: same racy set as the u64 encoding and the oracle."""
    tr = _random_batch(61, 40, max_blocks=4, max_warps=8, max_lanes=32, max_slots=12, n_words=500,
                       spaces=(0, 1), p_skip=0.3)
    o = oracle_set(tr)
    assert gpu_set(tr, compact=True, options=options) == o
    tr = tp.c1_tree_reduction(removed=8)
    assert gpu_set(tr, compact=True) == oracle_set(tr)


def test_compact_host_replay():
    from tracegen.format import to_c32
    h = hr()
    tr = tp.listing2(3, 4, 32)
    r32, rop = to_c32(tr)
    host = type("T", (), {"rec32": r32, "recop": rop, "kdesc": tr.kdesc, "warp_off": tr.warp_off,
                          "rec": None})()
    gmax, smem = h.trace_extent(tr)
    ck = h.Checker(gmax, smem)
    ck.replay_host(host)
    races, fl, _ = ck.report()
    assert [tuple(r) for r in races] == oracle_set(tr)[0]


@pytest.mark.parametrize("compact", [False, True])
def test_chunked_host_replay(compact, monkeypatch):
    """hr_replay_trace_host replays a kernel in block-range chunks as their
    records land (blocks are unordered by happens-before): force tiny chunks."""
    from tracegen.format import to_c32
    monkeypatch.setenv("HR_HOST_CHUNK_BYTES", "4096")
    h = hr()
    tr = _random_batch(81, 6, max_blocks=40, max_warps=4, max_lanes=32, max_slots=10, n_words=300,
                       spaces=(0, 1), grid=(37, 3, 32))
    tr2 = tp.listing2(33, 2, 32)
    for t in (tr, tr2):
        gmax, smem = h.trace_extent(t)
        ck = h.Checker(gmax, smem)
        if compact:
            r32, rop = to_c32(t)
            host = type("T", (), {"rec32": r32, "recop": rop, "kdesc": t.kdesc, "warp_off": t.warp_off,
                                  "rec": None})()
        else:
            host = t
        for _ in range(2):
            ck.reset()
            ck.replay_host(host)
            races, fl, _ = ck.report()
            assert ([tuple(r) for r in races], fl) == oracle_set(t)
        ck.close()


def test_soundness_at_scale():
    """SPEC.md:615 / PAPER.md:855 ("neither tool provided any false positives"):
    10,000 seeded random programs certified race-free by the oracle, replayed
    as one 10,000-kernel trace under both replay modes -> zero reports."""
    rng = random.Random(615)
    kernels = []
    while len(kernels) < 10000:
        t = tp.random_program(rng, max_blocks=2, max_warps=2, max_lanes=4, max_slots=6, n_words=3,
                              spaces=(0, 1), p_barrier=0.45)
        if oracle.check(t).races:
            continue
        b, w, l, sm, _ = (int(x) for x in t.kdesc[0, :5])
        k = tf.Kernel(b, w, l, sm)
        k.rows = [t.rec[int(t.warp_off[i]) * 32: int(t.warp_off[i + 1]) * 32].reshape(-1, 32) for i in range(b * w)]
        kernels.append(k)
    big = tf.make_trace(kernels)
    assert oracle.check(big).races == []
    for options in (16, 32):
        assert gpu_set(big, options=options) == ([], 0)


# ---- finite-history BASELINE detector (HR_OPT_FINITE_HISTORY) ----

FH = 128


def test_finite_history_misses_listing4_hirace_does_not():
    """with one reader record, thread 1's read of data[1] is
    evicted by thread 0's read, so thread 0's write finds no concurrent reader
    and the race "goes undetected"; HiRace's FSM keeps the summary.
    Rows run in program order inside a warp, so this eviction schedule is the
    one the replay executes."""
    tr = tp.listing4(1, 1, 4, 4)
    assert [r[3] for r in oracle_set(tr)[0]] == [1]
    assert [r[3] for r in gpu_set(tr)[0]] == [1]                 # HiRace: found
    assert gpu_set(tr, options=FH)[0] == []                      # finite history: missed
    big = tp.listing4(1, 8, 32, 256)                              # every word 1..253 racy
    assert len(gpu_set(big)[0]) == 253
    # inside a warp rows run in order, so the evicting read always comes second;
    # only words read by two warps (thread 32k and 32k-1) can escape eviction
    fh = {r[3] for r in gpu_set(big, options=FH)[0]}
    assert fh <= {32 * k for k in range(1, 8)}


def test_finite_history_is_sound_but_incomplete_on_c2():
    """Table II's shape: the finite-history detector never
    reports a word the oracle calls race-free, and misses some racy ones."""
    from tracegen import suite
    missed_traces = found_traces = 0
    for c in suite.suite():
        want = {(r.kernel, r.space, r.block, r.word) for r in oracle.check(c.trace).races}
        got = {tuple(r[:4]) for r in gpu_set(c.trace, options=FH)[0]}
        assert got <= want, c.name
        if want:
            if got:
                found_traces += 1
            else:
                missed_traces += 1
    assert found_traces > 0 and missed_traces > 0


@pytest.mark.parametrize("split", ["1", "2", "5"])
def test_split_helpers_same_result(split, monkeypatch):
    """Wide pooled replay with each simulated warp split over 2^split CUDA
    warps (clamped to 4 helpers and 32 warps per block): every word is still committed by
    one helper in record order, so the racy set is unchanged.  Mixed shared and
    global accesses, barriers, hot words, ragged warps."""
    monkeypatch.setenv("HR_SPLIT_LOG2", split)
    for seed, kw in ((121, dict(max_blocks=5, max_warps=4, max_lanes=32, max_slots=12, n_words=60,
                                spaces=(0, 1), p_barrier=0.25, p_skip=0.4)),
                     (122, dict(max_blocks=8, max_warps=8, max_lanes=32, max_slots=8, n_words=3,
                                spaces=(0, 1), p_skip=0.2)),
                     (123, dict(max_blocks=3, max_warps=32, max_lanes=32, max_slots=6, n_words=50,
                                spaces=(0, 1), p_barrier=0.3))):
        tr = _random_batch(seed, 12, **kw)
        assert gpu_set(tr, options=256) == oracle_set(tr)


def test_split_with_shards(monkeypatch):
    """Address shards (granule 9 and 5) combined with helper splitting: the
    union over shards equals the single-GPU set."""
    monkeypatch.setenv("HR_SPLIT_LOG2", "2")
    h = hr()
    tr = _random_batch(131, 16, max_blocks=4, max_warps=8, max_lanes=32, max_slots=10, n_words=3000,
                       spaces=(0, 1), p_barrier=0.2)
    gmax, smem = h.trace_extent(tr)
    full = oracle_set(tr)[0]
    for n, g in ((4, 9), (8, 5)):
        union = []
        for r in range(n):
            ck = h.Checker(gmax, smem, shard=(r, n), granule_log2=g, options=256)
            ck.replay(h.DeviceTrace.from_trace(tr))
            races, _, _ = ck.report()
            ck.close()
            union += [tuple(x) for x in races]
        assert sorted(union) == full


# ---- HR_OPT_SMEM32: 32-bit block-implicit shared-shadow words ----
S32 = 4096


@pytest.mark.parametrize("seed", range(3))
@pytest.mark.parametrize("options", [0, 16, 32, 256, 512])
def test_smem32_random_programs(seed, options):
    """Same racy set as the oracle with the clocks the 32-bit word can hold
    (bc 9 bits, wc 8 bits); shared and global words, full warps, barriers."""
    tr = _random_batch(300 + seed, 40, max_blocks=6, max_warps=8, max_lanes=32, max_slots=12,
                       n_words=40, spaces=(0, 1), p_barrier=0.25, p_skip=0.5)
    g, fl = gpu_set(tr, options=S32 | options)
    o, ofl = oracle_set(tr, bc_bits=9, wc_bits=8)
    assert g == o and fl == ofl
    assert any(r[1] == 1 for r in o)


def test_smem32_listings_c1_and_suite():
    from tracegen import suite
    for tr in (tp.listing1(2, 2, 32), tp.listing2(1, 32, 32), tp.listing4(1, 2, 32, 40),
               tp.c1_tree_reduction(removed=32), tp.c1_tree_reduction(removed=None)):
        assert gpu_set(tr, options=S32) == oracle_set(tr, bc_bits=9, wc_bits=8)
    for c in suite.suite():
        if c.trace.kdesc[:, 3].max() == 0:
            continue                                   # no shared memory in this case
        assert gpu_set(c.trace, options=S32) == oracle_set(c.trace, bc_bits=9, wc_bits=8), c.name


def test_smem32_clock_cap():
    """Past 511 block barriers the 32-bit word cannot tell epochs apart: the
    thread stops checking and the overflow flag is latched, exactly
    as the oracle with a 9-bit block clock does; the race before is kept."""
    ev = {(0, 0, 0): [tf.W(0, tf.SPACE_SHARED)] + [tf.SYNCTHREADS] * 600 + [tf.W(1, tf.SPACE_SHARED)],
          (0, 0, 1): [tf.W(0, tf.SPACE_SHARED)] + [tf.SYNCTHREADS] * 600 + [tf.W(1, tf.SPACE_SHARED)]}
    tr = tp.from_thread_events(1, 1, 2, ev, smem_words=2)
    g, fl = gpu_set(tr, options=S32)
    o, ofl = oracle_set(tr, bc_bits=9, wc_bits=8)
    assert g == o and fl == ofl == hr().HR_F_CLOCK_OVERFLOW
    assert [r[3] for r in g] == [0]
    # the 64-bit word keeps checking: both words are racy
    assert [r[3] for r in gpu_set(tr)[0]] == [0, 1]


def test_smem32_with_finite_history_rejected():
    h = hr()
    with pytest.raises(Exception):
        h.Checker(64, 64, options=S32 | h.HR_OPT_FINITE_HISTORY)


# ---- HR_OPT_LAZY_RESET: epoch-tagged global shadow, no per-kernel memset (§8(f)-4) ----
LAZY = 8192


def _concat(traces):
    """One multi-kernel trace from single-kernel traces (kernel boundaries between)."""
    kernels = []
    for t in traces:
        for k in range(t.kdesc.shape[0]):
            blocks, warps, lanes, smem, woi = (int(x) for x in t.kdesc[k, :5])
            kk = tf.Kernel(blocks, warps, lanes, smem)
            kk.rows = [t.rec[int(t.warp_off[woi + w]) * 32: int(t.warp_off[woi + w + 1]) * 32].reshape(-1, 32)
                       for w in range(blocks * warps)]
            kernels.append(kk)
    return tf.make_trace(kernels)


@pytest.mark.parametrize("options", [0, 16, 32, 256, 512, 4096])
def test_lazy_reset_many_kernels(options):
    """300 and 40 kernels reusing the same words: tags wrap every 15 kernels
    (real reset), stale words of earlier kernels must read as INIT."""
    tr = _random_batch(11, 300, max_blocks=2, max_warps=2, max_lanes=2, max_slots=5, n_words=2, spaces=(0, 1))
    assert gpu_set(tr, options=LAZY | options) == oracle_set(tr)
    tr = _random_batch(12, 40, max_blocks=6, max_warps=8, max_lanes=32, max_slots=12, n_words=40,
                       spaces=(0, 1), p_barrier=0.25, p_skip=0.5)
    assert gpu_set(tr, options=LAZY | options) == oracle_set(tr)


def test_lazy_reset_suite_and_c1():
    from tracegen import suite
    for c in suite.suite():
        assert gpu_set(c.trace, options=LAZY) == oracle_set(c.trace), c.name
    tr = tp.c1_tree_reduction(removed=16)
    assert gpu_set(tr, options=LAZY) == oracle_set(tr)


def test_lazy_reset_overflow_scan_skips_stale_words():
    """Kernel A leaves RACE words in the global shadow; kernel B (other words)
    overflows the ring, so the report scans B's shadow: A's words carry A's
    tag and must not come back as B's races."""
    a = tp.from_thread_events(1, 1, 2, {(0, 0, 0): [tf.W(1000)], (0, 0, 1): [tf.W(1000)]})   # kernel 0: word 1000
    b = tp.listing2(4, 8, 32)                         # many racy words in kernel 1
    tr = _concat([a, b])
    want, _ = oracle_set(tr)
    assert [r[3] for r in want if r[0] == 0] == [1000] and any(r[0] == 1 for r in want)
    assert all(r[3] != 1000 for r in want if r[0] == 1)
    g, fl = gpu_set(tr, options=LAZY, ring_capacity=8)
    assert fl & hr().HR_F_RING_OVERFLOW
    assert g == want


def test_lazy_reset_rejected_with_double_shadow():
    h = hr()
    with pytest.raises(Exception):
        h.Checker(64, 0, options=LAZY | h.HR_OPT_DOUBLE_SHADOW)


def test_lazy_reset_repeated_replays_device_and_host():
    """The bench pattern: the same multi-kernel trace replayed again and again
    on one ctx (tags wrap several times), from device memory, from host
    buffers (chunked) and from the PACKED encoding: every report equals the
    oracle's."""
    h = hr()
    tr = _random_batch(21, 7, max_blocks=6, max_warps=8, max_lanes=32, max_slots=12, n_words=40,
                       spaces=(0, 1), p_barrier=0.25, p_skip=0.5)
    want, _ = oracle_set(tr)
    gmax, smem = h.trace_extent(tr)
    ck = h.Checker(gmax, smem, options=LAZY)
    dt = h.DeviceTrace.from_trace(tr)
    packed_host = ck.pack(dt).to_host()
    for i in range(12):                                   # 84 kernels: 5 tag wraps
        ck.reset()
        if i % 3 == 0:
            ck.replay(dt)
        elif i % 3 == 1:
            ck.replay_host(tr)
        else:
            ck.replay_host(packed_host)
        races, fl, _ = ck.report()
        assert [tuple(r) for r in races] == want and fl == 0, i
    ck.close()


# ---- hr_report_async / hr_report_collect: a13 on the device ----
def _async_vs_sync(tr, **kw):
    h = hr()
    gmax, smem = h.trace_extent(tr)
    ck = h.Checker(gmax, smem, **kw)
    dt = h.DeviceTrace.from_trace(tr)
    ck.reset(); ck.replay(dt); ck.report_async()
    a_raw, a_fl = ck.collect_raw()
    sync_raw, sync_fl = ck.report_raw()               # same ring: byte-identical, witnesses included
    ck.close()
    return sync_raw, sync_fl, a_raw, a_fl


def test_report_async_matches_sync_and_oracle():
    from tracegen import suite
    cases = [c.trace for c in suite.suite()[::7]] + [
        tp.listing2(64, 8, 32),                        # > 4096 races
        tp.listing1(1, 1, 1),                          # no race
        _random_batch(5, 30, max_blocks=6, max_warps=8, max_lanes=32, max_slots=12, n_words=40,
                      spaces=(0, 1), p_barrier=0.25, p_skip=0.5)]
    for tr in cases:
        s_raw, s_fl, a_raw, a_fl = _async_vs_sync(tr)
        assert a_raw.tobytes() == s_raw.tobytes() and a_fl == s_fl
        assert [(int(r["kernel"]), int(r["space"]), int(r["block"]), int(r["word"]), int(r["scope"]))
                for r in a_raw] == oracle_set(tr)[0]


def test_report_async_ring_overflow_falls_back():
    tr = tp.listing2(4, 8, 32)
    s_raw, s_fl, a_raw, a_fl = _async_vs_sync(tr, ring_capacity=8)
    assert a_fl & hr().HR_F_RING_OVERFLOW
    assert a_raw.tobytes() == s_raw.tobytes()
    assert [(int(r["kernel"]), int(r["space"]), int(r["block"]), int(r["word"]), int(r["scope"]))
            for r in a_raw] == oracle_set(tr)[0]


def test_report_async_c5_planted_repeated():
    """The bench pattern: several enqueued steps, each replay followed by an
    async report, one collect at the end = the planted set (closed form)."""
    from tracegen import c5
    h = hr()
    lb = 8
    rec, woff, kd = c5.gpu_trace(lb)
    dt = h.DeviceTrace(rec, woff, kd)
    ck = h.Checker(c5.total_words(lb), 0, ring_capacity=1 << 16, options=h.HR_OPT_LAZY_RESET)
    for _ in range(4):
        ck.reset(); ck.replay(dt); ck.report_async()
    raw, fl = ck.collect_raw()
    ck.close()
    assert fl == 0
    assert [(int(r["word"]), int(r["scope"])) for r in raw] == c5.planted(lb)


@pytest.mark.parametrize("lb", [10, 12, 15])
def test_report_async_graph_paths(lb):
    """hr_report_async is one CUDA graph: up to 8192 ring records take the
    one-CTA small-set kernel, more take the conditional full-capacity sort (C5
    at 2^lb blocks plants 2^lb racy words, with one or two ring records each:
    2^12 fit the small path, 2^15 do not).  Both equal the
    synchronous report byte for byte and the planted set (closed form); the
    launch count shows which path ran."""
    from tracegen import c5
    h = hr()
    rec, woff, kd = c5.gpu_trace(lb)
    dt = h.DeviceTrace(rec, woff, kd)
    ck = h.Checker(c5.total_words(lb), 0, ring_capacity=1 << 16, options=h.HR_OPT_LAZY_RESET)
    launches = []
    for _ in range(2):
        ck.reset(); ck.replay(dt)
        h.hr_launch_count(ck.ctx)
        ck.report_async()
        a_raw, a_fl = ck.collect_raw()
        launches.append(h.hr_launch_count(ck.ctx))
    s_raw, s_fl = ck.report_raw()
    ck.close()
    assert a_raw.tobytes() == s_raw.tobytes() and a_fl == s_fl == 0
    assert [(int(r["word"]), int(r["scope"])) for r in a_raw] == c5.planted(lb)
    # spill scan + small-set kernel; the IF body adds its keys / sort / heads / scan / emit kernels
    assert launches[0] == launches[1]
    assert (launches[0] == 2) == (lb <= 12), launches


def test_report_async_small_out_cap_and_runs():
    """Small-set path with several records per address (scope upgrades across
    kernels of one ctx are separate addresses; within a kernel RACE_BLOCK then
    RACE_GRID records merge to the widest scope) and an hr_report_async_to
    buffer smaller than the set: hdr[0] is the full count, the first out_cap
    records are the sorted prefix."""
    import torch
    h = hr()
    tr = _random_batch(77, 60, max_blocks=6, max_warps=8, max_lanes=32, max_slots=12, n_words=24,
                       spaces=(0, 1), p_barrier=0.2, p_skip=0.3)
    want = oracle_set(tr)[0]
    assert len(want) > 8
    gmax, smem = h.trace_extent(tr)
    ck = h.Checker(gmax, smem)
    dt = h.DeviceTrace.from_trace(tr)
    ck.reset(); ck.replay(dt); ck.report_async()
    a_raw, _ = ck.collect_raw()
    assert [(int(r["kernel"]), int(r["space"]), int(r["block"]), int(r["word"]), int(r["scope"]))
            for r in a_raw] == want
    cap = 5
    out = torch.zeros(cap * 24, dtype=torch.uint8, device="cuda")
    hdr = torch.zeros(4, dtype=torch.int32, device="cuda")
    for _ in range(3):                     # alternating targets: both cached report graphs
        out.zero_(); hdr.zero_()
        h.hr_report_async_to(ck.ctx, out.data_ptr(), cap, hdr.data_ptr())
        torch.cuda.synchronize()
        got = np.frombuffer(out.cpu().numpy().tobytes(), dtype=a_raw.dtype)
        assert int(hdr[0]) == len(want)
        assert got.tobytes() == a_raw[:cap].tobytes()
        ck.report_async()
        b_raw, _ = ck.collect_raw()
        assert b_raw.tobytes() == a_raw.tobytes()
    ck.close()


# ---- HR_OPT_BSERIAL: block-serial pooled replay (hr_bserial.cuh) ----
BS = 16384 | 32                                      # forced, with the pooled kernel choice


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("extra", [0, 1, 4096, 8192, 2048])
def test_bserial_random_programs(seed, extra):
    """Barriers, __syncwarp, shared and global words, full and ragged warps,
    up to 8 warps per block: the block-serial walk gives the oracle's set."""
    tr = _random_batch(400 + seed, 40, max_blocks=6, max_warps=8, max_lanes=32, max_slots=12, n_words=40,
                       spaces=(0, 1), p_barrier=0.25, p_skip=0.5)
    g, fl = gpu_set(tr, options=BS | extra)
    bc, wc = (9, 8) if extra == 4096 else (16, 16)
    o, ofl = oracle_set(tr, bc_bits=bc, wc_bits=wc)
    assert g == o and fl == ofl
    tr = _random_batch(500 + seed, 200, max_blocks=2, max_warps=4, max_lanes=3, max_slots=6, n_words=3,
                       spaces=(0, 1))
    assert gpu_set(tr, options=BS | extra) == oracle_set(tr)


def test_bserial_suite_listings_and_shards():
    from tracegen import suite
    for c in suite.suite():
        assert gpu_set(c.trace, options=BS) == oracle_set(c.trace), c.name
    for tr in (tp.listing1(64, 8, 32), tp.listing2(3, 4, 32), tp.listing4(1, 2, 32, 40),
               tp.c1_tree_reduction(removed=32)):
        assert gpu_set(tr, options=BS) == oracle_set(tr)
    h = hr()
    tr = _random_batch(51, 20, max_blocks=4, max_warps=4, max_lanes=32, max_slots=10, n_words=3000, spaces=(0, 1))
    gmax, smem = h.trace_extent(tr)
    full, _ = gpu_set(tr)
    for n, g in ((2, 9), (8, 3), (8, 0)):
        union = []
        for r in range(n):
            ck = h.Checker(gmax, smem, shard=(r, n), granule_log2=g, options=BS)
            ck.replay(h.DeviceTrace.from_trace(tr))
            races, _, _ = ck.report()
            ck.close()
            union += [tuple(x) for x in races]
        assert sorted(union) == full


def test_bserial_clock_overflow():
    ev = {(0, 0, 0): [tf.W(0)] + [tf.SYNCTHREADS] * 4 + [tf.W(1)],
          (0, 0, 1): [tf.W(0)] + [tf.SYNCTHREADS] * 4 + [tf.W(1)]}
    tr = tp.from_thread_events(1, 1, 2, ev)
    g, fl = gpu_set(tr, bc_bits=2, wc_bits=30, options=BS)
    o, ofl = oracle_set(tr, bc_bits=2, wc_bits=30)
    assert g == o and fl == ofl == hr().HR_F_CLOCK_OVERFLOW


def test_bserial_c5_planted():
    from tracegen import c5
    h = hr()
    lb = 8
    for n in (1, 8):
        for r in ((0, n - 1) if n > 1 else (0,)):
            rec, woff, kd = c5.gpu_trace(lb, rank=r, nshard=n)
            ck = h.Checker(c5.total_words(lb), 0, ring_capacity=1 << 16, shard=(r, n), options=BS | h.HR_OPT_LAZY_RESET)
            ck.replay(h.DeviceTrace(rec, woff, kd))
            raw, fl = ck.report_raw()
            ck.close()
            from paper_2401_04701_b200.multigpu import shard_owner
            want = [(w, sc) for w, sc in c5.planted(lb) if n == 1 or shard_owner(w >> 3, n) == r]
            assert fl == 0 and [(int(x["word"]), int(x["scope"])) for x in raw] == want


# ---- representative threads (hr_set_representatives) ----
def _only_representatives(tr, bs, ws):
    """The trace with the access records of non-representative threads turned
    into NOPs (their barrier records stay): what the oracle must see."""
    import copy
    out = copy.copy(tr)
    rec = tr.rec.copy()
    nop = np.uint64(3 << 62)
    for k in range(tr.kdesc.shape[0]):
        blocks, warps, lanes, smem, woi = (int(x) for x in tr.kdesc[k, :5])
        for gw in range(blocks * warps):
            b, w = gw // warps, gw % warps
            if (bs <= 1 or b % bs == 0) and (ws <= 1 or w % ws == 0):
                continue
            seg = rec[int(tr.warp_off[woi + gw]) * 32: int(tr.warp_off[woi + gw + 1]) * 32]
            seg[(seg >> np.uint64(62)) != 3] = nop
    out.rec = rec
    return out


@pytest.mark.parametrize("reps", [(2, 1), (1, 2), (3, 2), (1, 1)])
@pytest.mark.parametrize("options", [0, 16, 32, 256, 512, 16384 | 32])
def test_representatives_equal_the_restricted_trace(reps, options):
    tr = _random_batch(600, 30, max_blocks=6, max_warps=8, max_lanes=32, max_slots=12, n_words=40,
                       spaces=(0, 1), p_barrier=0.25, p_skip=0.5)
    g = [tuple(r) for r in hr().check_trace(tr, options=options, representatives=reps)[0]]
    want, _ = oracle_set(_only_representatives(tr, *reps))
    assert g == want
    if reps != (1, 1):
        assert len(want) < len(oracle_set(tr)[0])          # the filter drops races, by design


def test_representatives_suite():
    from tracegen import suite
    for c in suite.suite()[::5]:
        g = [tuple(r) for r in hr().check_trace(c.trace, representatives=(2, 2))[0]]
        assert g == oracle_set(_only_representatives(c.trace, 2, 2))[0], c.name


# ---- shared rows (hr__check_shared_row: wide and narrow row kernels, C32 and u64 records) ----
def _shared_rows_trace(seed, n_kernels=6, n_rows=40, smem=1024, private=False):
    """Full warps whose rows are mostly "shared rows" (32 strictly increasing
    shared words, any kinds), with repeated rows (the same word twice in a row
    per lane), block barriers at common row indices, and some global or
    non-increasing rows in between (pairs broken off).  private: each shared
    word belongs to one lane of one warp (race-free shared space)."""
    rng = np.random.default_rng(seed)
    kernels = []
    for _ in range(n_kernels):
        blocks, warps = int(rng.integers(1, 5)), int(rng.integers(1, 9))
        kinds = rng.choice([0, 1, 2, 3], size=n_rows, p=[0.72, 0.1, 0.08, 0.1])   # shared / global / shuffled / barrier
        rows = np.zeros((blocks * warps, n_rows, 32), dtype=np.uint64)
        for w in range(blocks * warps):
            prev = None
            for i in range(n_rows):
                if kinds[i] == 3:
                    rows[w, i, :] = tf.SYNCTHREADS
                    prev = None
                    continue
                if prev is not None and rng.random() < 0.3:
                    words = prev                                           # same words as the last row
                elif private:
                    words = (w % warps) * 128 + 32 * int(rng.integers(0, 4)) + np.arange(32)
                else:
                    s = int(rng.integers(1, 4))
                    words = int(rng.integers(0, smem - 32 * s)) + s * np.arange(32)
                if kinds[i] == 2 and not private:
                    words = rng.permutation(words)                         # not increasing: general path
                ops = rng.choice([0, 1, 2], size=32, p=[0.7, 0.2, 0.1])
                space = 0 if kinds[i] == 1 else 1
                rows[w, i, :] = [tf.encode(int(o), space, int(x)) for o, x in zip(ops, words)]
                if private and kinds[i] == 2:
                    rows[w, i, rng.random(32) < 0.3] = tf.NOP           # partial row: general path
                prev = words if kinds[i] == 0 else None
        kernels.append(tf.kernel_from_rows(blocks, warps, 32, rows, smem_words=smem))
    return tf.make_trace(kernels)


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("options", [0, 512, 65536])
def test_shared_rows_paired(seed, options):
    """Runs of shared rows (the specialised shared-row check) in the wide and
    the narrow row kernel = the oracle: racy and race-free words, the same
    words in consecutive rows, runs broken by barriers, global rows, shuffled
    or partial rows (general path)."""
    tr = _shared_rows_trace(900 + seed)
    o = oracle_set(tr)
    assert gpu_set(tr, compact=True, options=options) == o
    assert gpu_set(tr, options=options) == o
    assert len(o[0]) > 0
    tr = _shared_rows_trace(950 + seed, private=True)
    o = oracle_set(tr)
    assert gpu_set(tr, compact=True, options=options) == o
    assert all(r[1] == 0 for r in o[0])                 # only the global rows race
