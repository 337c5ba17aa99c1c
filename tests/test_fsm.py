"""The generated FSM table (product, paper_2401_04701_b200/fsm) against the
paper's named transitions, the Fig. 1 machine, structural properties, and —
the parity gate — the CPU oracle over every happens-before-consistent commit
order of every address of random programs (the
"Murphi" exhaustive check of PAPER.md:569 replaced by differential search).
"""
import os
import random

import pytest

import oracle
from paper_2401_04701_b200.fsm import generate as G
from tests import helpers as H
from tracegen import programs as tp

TABLE, FLAGS, MC = G.build_table()
R, W, A = G.K_R, G.K_W, G.K_A
US, WS, BS = G.S_US, G.S_WS, G.S_BS
S, WP, B, GL = G.T_S, G.T_W, G.T_B, G.T_G
CODE = {name: c for c, name in MC.names.items()}
RACES = (G.RACE_BLOCK_CODE, G.RACE_GRID_CODE)


def nxt(state, m, s, t):
    return TABLE[(CODE[state] << 6) | (m << 4) | (s << 2) | t]


def is_race(code):
    return code in RACES


def test_size_and_encoding():
    # 5 bits of state -> at most 32 states
    assert MC.n_states <= 32
    assert MC.n_states == 22
    assert CODE["INIT"] == 0 and len(TABLE) == 2048 and len(FLAGS) == 32


def test_committed_table_is_current():
    with open(G.INC_PATH) as f:
        assert f.read() == G.render_inc(TABLE, FLAGS, MC)


def test_scenario1_transitions():
    """PAPER.md:464-469 (Scenario 1, Fig. 1)."""
    for s, t in ((US, S), (US, GL), (BS, B)):
        assert MC.names[TABLE[(0 << 6) | (R << 4) | (s << 2) | t]] == "READ"   # INIT -R*-> READ
    assert MC.names[nxt("READ", R, US, GL)] == "GREAD"     # "advances the state to GREAD"
    for s in (US,):
        for t in (S, WP, B, GL):
            assert is_race(nxt("GREAD", W, s, t))          # "W* arc ... to RACE"
    assert MC.names[nxt("READ", W, US, S)] == "WRITE"      # W_S "same-thread write"
    assert is_race(nxt("WRITE", R, US, GL))                # "any read or write access by a
    assert is_race(nxt("WRITE", W, US, GL))                #  different thread is a race"


def test_scenario2_transitions():
    """PAPER.md:545-558 (Scenario 2, Fig. 4)."""
    assert MC.names[nxt("READ", R, US, B)] == "BREAD"      # R{Us,B}
    assert MC.names[nxt("BREAD", R, US, B)] == "BREAD"     # "remains in the BRead state"
    assert MC.names[nxt("BREAD", R, US, GL)] == "GREAD"    # R{*,G}
    for s, t in ((US, S), (US, B), (US, GL), (BS, S), (BS, B)):
        assert is_race(nxt("GREAD", W, s, t))              # W{*,*} from GRead
    assert MC.names[nxt("BREAD", W, BS, S)] == "WRITE"     # W{Bs,S}
    assert MC.names[nxt("BREAD", W, BS, B)] == "WRITE"     # W{Bs,B}
    assert is_race(nxt("WRITE", R, US, GL))                # T110 reads -> Race
    assert is_race(nxt("BREAD", W, US, B))                 # unsynchronised write after block reads


def test_race_absorbing_and_scope_monotone():
    for m in range(3):
        for s in range(3):
            for t in range(4):
                if not G.feasible(s, t):
                    continue
                assert TABLE[(31 << 6) | (m << 4) | (s << 2) | t] == 31
                assert TABLE[(30 << 6) | (m << 4) | (s << 2) | t] == (31 if t == GL else 30)


def test_init_ignores_label():
    for m in range(3):
        vals = {TABLE[(m << 4) | (s << 2) | t] for s in range(3) for t in range(4)}
        assert len(vals) == 1 and not is_race(vals.pop())


def test_totality():
    for c in MC.codes():
        for m in range(3):
            for s in range(4):
                for t in range(4):
                    assert TABLE[(c << 6) | (m << 4) | (s << 2) | t] in MC.codes()


def test_independent_sync_bits():
    """hr__check_shared_row sets the two sync bits independently (bit 1: block
    epoch differs, bit 0: warp epoch differs): index 3 must act as Bs (Bs
    dominates Ws) and Ws with a Block relation as Us (a warp
    clock says nothing across warps), so the table resolves the label."""
    for c in MC.codes():
        for m in range(3):
            row = lambda s, t: TABLE[(c << 6) | (m << 4) | (s << 2) | t]
            for t in range(3):
                assert row(3, t) == row(2, t)
            assert row(3, 3) == row(0, 3)
            assert row(1, 2) == row(0, 2)


def test_fig1_restriction_is_five_states():
    """Fig. 1: reads/writes, no barriers, relations
    Self/Global -> exactly INIT, READ, GREAD, WRITE, RACE, with unmentioned
    transitions self-loops (caption)."""
    labels = [(m, US, t) for m in (R, W) for t in (S, GL)]
    mc = G.Machine(labels=labels, split_race=False)
    assert mc.n_states == 5
    names = set(mc.names.values())
    assert {"INIT", "READ", "GREAD", "WRITE"} <= names
    inv = {v: k for k, v in mc.code.items()}
    code = {n: c for c, n in mc.names.items()}
    race = [c for c, n in mc.names.items() if n.startswith("RACE")][0]
    # the figure's arcs (Scenario 1): everything else is a self loop
    arcs = {("INIT", R, S): "READ", ("INIT", R, GL): "READ", ("INIT", W, S): "WRITE",
            ("INIT", W, GL): "WRITE", ("READ", R, GL): "GREAD", ("READ", W, S): "WRITE",
            ("READ", W, GL): race, ("GREAD", W, S): race, ("GREAD", W, GL): race,
            ("WRITE", R, GL): race, ("WRITE", W, GL): race}
    for src in ("INIT", "READ", "GREAD", "WRITE"):
        for m in (R, W):
            for t in (S, GL):
                want = arcs.get((src, m, t), src)
                want = want if isinstance(want, int) else code[want]
                assert mc.next_code(code[src], m, US, t) == want, (src, m, t)


def test_insensitive_flags():
    # GREAD/GATOMIC/RACE_GRID: label-insensitive closure
    for n in ("GREAD", "GATOMIC", "RACE_GRID"):
        assert FLAGS[CODE[n]] & G.FLAG_INSENSITIVE
    assert FLAGS[CODE["RACE_BLOCK"]] & G.FLAG_BLOCK_ONLY
    assert not FLAGS[CODE["RACE_BLOCK"]] & G.FLAG_INSENSITIVE
    for n in ("READ", "WRITE", "BREAD", "ATOMIC"):
        assert not FLAGS[CODE[n]] & (G.FLAG_INSENSITIVE | G.FLAG_BLOCK_ONLY)


def test_stale_probe_exit_is_safe():
    """hr_device.cuh takes the insensitive exit on a possibly stale L1 value:
    valid iff every state reachable from it is also a no-op for that kind."""
    def reach(c):
        seen, st = {c}, [c]
        while st:
            x = st.pop()
            for m in range(3):
                for s in range(3):
                    for t in range(4):
                        if G.feasible(s, t):
                            y = TABLE[(x << 6) | (m << 4) | (s << 2) | t]
                            if y not in seen:
                                seen.add(y)
                                st.append(y)
        return seen
    n = 0
    for c in MC.codes():
        if not FLAGS[c] & G.FLAG_INSENSITIVE:
            continue
        for m in range(3):
            if TABLE[(c << 6) | (m << 4)] != c:
                continue
            for y in reach(c):
                assert FLAGS[y] & G.FLAG_INSENSITIVE
                assert all(TABLE[(y << 6) | (m << 4) | (s << 2) | t] == y
                           for s in range(3) for t in range(4) if G.feasible(s, t))
            n += 1
    assert n >= 3


def _differential(table, programs, cap=2000):
    """For every address and every HB-consistent commit order: Algorithm 1 over
    ``table`` ends in RACE (with the oracle's scope) iff the oracle says racy.
    Returns (orders checked, mismatches)."""
    n_orders, bad = 0, []
    for tr in programs:
        res = oracle.check(tr, mode=oracle.PAIRWISE)
        want = {(r.kernel, r.space, r.block, r.word): r.scope for r in res.races}
        for key, accs in H.accesses_by_address(tr).items():
            exp = want.get(key, 0)
            for order in H.linear_extensions(accs, cap=cap):
                n_orders += 1
                final, trail = H.run_word(table, order)
                got = H.scope_of(final)
                if got != exp:
                    bad.append((tr, key, order, got, exp))
                    break
    return n_orders, bad


def _family(seed, n, **kw):
    rng = random.Random(seed)
    return [tp.random_program(rng, **kw) for _ in range(n)]


def test_differential_small_family():
    """S:612 family: <=2 blocks x <=2 warps x <=2 lanes, <=3 events/thread,
    <=2 addresses, kinds R/W/A, both barrier types."""
    progs = _family(11, 1500, max_blocks=2, max_warps=2, max_lanes=2, max_slots=4,
                    n_words=2, spaces=(0, 1))
    n, bad = _differential(TABLE, progs)
    assert not bad, bad[:1]
    assert n > 20000


def test_differential_wider_grids():
    progs = _family(12, 300, max_blocks=3, max_warps=3, max_lanes=3, max_slots=6,
                    n_words=2, p_skip=0.5)
    n, bad = _differential(TABLE, progs, cap=500)
    assert not bad, bad[:1]


def test_fault_injection_detected():
    """GREAD-on-write rerouted to WRITE must be caught."""
    t = bytearray(TABLE)
    g, wcode = CODE["GREAD"], CODE["WRITE"]
    for s in range(4):
        for r in range(4):
            t[(g << 6) | (W << 4) | (s << 2) | r] = wcode
    progs = _family(13, 400, max_blocks=2, max_warps=2, max_lanes=2, max_slots=4, n_words=1)
    _, bad = _differential(bytes(t), progs, cap=50)
    assert bad


def test_listing4_every_schedule_races():
    """"any number of reads and any scheduling ... must
    eventually reach the Race state"."""
    tr = tp.listing4(1, 1, 6, 6)
    acc = H.accesses_by_address(tr)
    for key, accs in acc.items():
        word = key[3]
        for order in H.linear_extensions(accs):
            final, _ = H.run_word(TABLE, order)
            assert (final in RACES) == (1 <= word <= 3)


@pytest.mark.slow
def test_differential_large():
    progs = _family(21, 20000, max_blocks=2, max_warps=2, max_lanes=2, max_slots=4,
                    n_words=2, spaces=(0, 1))
    n, bad = _differential(TABLE, progs, cap=5000)
    assert not bad, bad[:1]


# ---- race-class projections ----

CLASS_MACHINES = G.class_machines()


def test_class_projection_sizes_and_inc():
    sizes = {name: mc.n_states for name, _, _, mc in CLASS_MACHINES}
    assert sizes == {"WW": 3, "RW": 21, "AW": 21, "AR": 21}
    with open(G.CLASSES_INC_PATH) as f:
        assert f.read() == G.render_classes_inc(CLASS_MACHINES)


def _class_differential(programs, cap=500):
    n, bad = 0, []
    for tr in programs:
        res = oracle.check(tr, mode=oracle.PAIRWISE)
        want = {(r.kernel, r.space, r.block, r.word): c for r, c in zip(res.races, res.classes)}
        for key, accs in H.accesses_by_address(tr).items():
            exp = want.get(key, 0)
            for order in H.linear_extensions(accs, cap=cap):
                got = 0
                for bit, (name, kinds, table, _) in enumerate(CLASS_MACHINES):
                    sub = [a for a in order if a[4] in kinds]
                    final, _ = H.run_word(table, sub)
                    if final == G.RACE_BLOCK_CODE:
                        got |= 1 << bit
                n += 1
                if got != exp:
                    bad.append((key, order, got, exp))
                    break
    return n, bad


def test_class_projections_match_oracle():
    """Each projection enters RACE over every HB-consistent order iff the
    oracle finds a race pair of its class (schedule-independent classes)."""
    progs = _family(31, 1200, max_blocks=2, max_warps=2, max_lanes=2, max_slots=4, n_words=2,
                    spaces=(0, 1))
    n, bad = _class_differential(progs)
    assert not bad, bad[:1]
    assert n > 15000
