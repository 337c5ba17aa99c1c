"""Per-pair race classes: hr_race_classes on the GPU equals
the oracle's class masks (bit0 W-W, bit1 R-W, bit2 A-W, bit3 A-R) for every
racy address, bit for bit."""
import random

import pytest

import oracle
from tracegen import c4, programs as tp, stencil, suite
from tracegen import format as tf

pytestmark = pytest.mark.gpu


def hr():
    from paper_2401_04701_b200 import hirace
    return hirace


def gpu_classes(trace, **kw):
    h = hr()
    gmax, smem = h.trace_extent(trace)
    ck = h.Checker(gmax, smem, ring_capacity=1 << 22, **kw)
    dt = h.DeviceTrace.from_trace(trace)
    ck.replay(dt)
    raw, flags = ck.report_raw()
    cls = ck.classes(dt, raw)
    ck.close()
    return ([(int(r["kernel"]), int(r["space"]), int(r["block"]), int(r["word"]), int(r["scope"])) for r in raw],
            [int(c) for c in cls])


def oracle_classes(trace):
    res = oracle.check(trace)
    return [tuple(r) for r in res.races], list(res.classes)


def test_listings_classes():
    for tr in (tp.listing1(2, 2, 32), tp.listing2(2, 4, 32), tp.listing4(1, 4, 32, 100)):
        assert gpu_classes(tr) == oracle_classes(tr)


def test_c2_suite_classes():
    n = 0
    for c in suite.suite():
        want = oracle_classes(c.trace)
        if want[0]:
            assert gpu_classes(c.trace) == want, c.name
            n += 1
    assert n > 250


@pytest.mark.parametrize("seed", range(3))
def test_random_programs_classes(seed):
    rng = random.Random(900 + seed)
    kernels = []
    for _ in range(40):
        t = tp.random_program(rng, max_blocks=4, max_warps=4, max_lanes=32, max_slots=10, n_words=12,
                              spaces=(0, 1), p_skip=0.4)
        b, w, l, sm, _ = (int(x) for x in t.kdesc[0, :5])
        k = tf.Kernel(b, w, l, sm)
        k.rows = [t.rec[int(t.warp_off[i]) * 32: int(t.warp_off[i + 1]) * 32].reshape(-1, 32) for i in range(b * w)]
        kernels.append(k)
    tr = tf.make_trace(kernels)
    want = oracle_classes(tr)
    assert len(want[0]) > 20
    assert {c for c in want[1]} - {0} and gpu_classes(tr) == want


def test_c1_c3_c4_classes():
    for tr in (tp.c1_tree_reduction(removed=16), stencil.stencil_trace(removed=20, n=128), c4.Graph(16).trace(True)):
        assert gpu_classes(tr) == oracle_classes(tr)
