"""Online instrumentation (include/hr_device.cuh used inside real kernels,
include/hr_bench.h): the instrumented C1 / C3 / C4 kernels report exactly the
oracle's racy set on the traces tracegen generates for the same kernels, and
the plain kernels compute the right values."""
import numpy as np
import pytest

import oracle
from tracegen import c4, programs as tp, stencil

pytestmark = pytest.mark.gpu


def mods():
    from paper_2401_04701_b200 import hirace, online
    return hirace, online


def _races(raw):
    return [(int(r["kernel"]), int(r["space"]), int(r["block"]), int(r["word"]), int(r["scope"])) for r in raw]


@pytest.mark.parametrize("removed", [None, "load", 128, 32, 16, 4, 1])
def test_c1_online_matches_oracle(removed):
    import torch
    hr, on = mods()
    data = torch.arange(8 * 256 + 8, dtype=torch.int32, device="cuda")
    ck = hr.Checker(8 * 256 + 8, 256)
    on.c1(ck.ctx, data, True, removed=removed)
    raw, flags = ck.report_raw()
    want = oracle.check(tp.c1_tree_reduction(removed=removed))
    assert _races(raw) == [tuple(r) for r in want.races] and flags == 0
    if removed is None:
        # the plain kernel reduces each round's 256 inputs
        d2 = torch.arange(8 * 256 + 8, dtype=torch.int32, device="cuda")
        on.c1(None, d2, False, removed=None)
        torch.cuda.synchronize()
        exp = [sum(range(r * 256, (r + 1) * 256)) for r in range(8)]
        assert d2[2048:].tolist() == exp


@pytest.mark.parametrize("removed", [None, 32, 8, "load"])
def test_c1_transparent_wrapper_matches_oracle(removed):
    """hr_array<T> (PAPER.md:676-678 wrapper class) instruments plain-looking
    code; the racy set equals the oracle's on the C1 trace."""
    import torch
    hr, on = mods()
    data = torch.arange(8 * 256 + 8, dtype=torch.int32, device="cuda")
    ck = hr.Checker(8 * 256 + 8, 256)
    on.c1_array(ck.ctx, data, removed=removed)
    raw, flags = ck.report_raw()
    want = oracle.check(tp.c1_tree_reduction(removed=removed))
    assert _races(raw) == [tuple(r) for r in want.races] and flags == 0
    if removed is None:
        torch.cuda.synchronize()
        assert data[2048:].tolist() == [sum(range(r * 256, (r + 1) * 256)) for r in range(8)]


@pytest.mark.parametrize("n,removed", [(128, 20), (128, None), (512, 20)])
def test_c3_online_matches_oracle(n, removed):
    import torch
    hr, on = mods()
    data = torch.randint(0, 100, (2 * n * n,), dtype=torch.int32, device="cuda")
    ck = hr.Checker(2 * n * n, 648, ring_capacity=1 << 20)
    on.c3(ck.ctx, data, True, n=n, removed=removed)
    raw, flags = ck.report_raw()
    want = oracle.check(stencil.stencil_trace(removed=removed, n=n))
    assert _races(raw) == [tuple(r) for r in want.races] and flags == 0


@pytest.mark.parametrize("racy", [True, False])
def test_c4_online_matches_oracle(racy):
    import torch
    hr, on = mods()
    g = c4.Graph(16)
    dev = on.C4Device(g)
    data = torch.full((g.n + 1024,), -1, dtype=torch.int32, device="cuda")
    data[g.n:] = 0
    ck = hr.Checker(g.n + 1024, 0, ring_capacity=1 << 20)
    dev.run(ck.ctx, data, True, racy)
    raw, flags = ck.report_raw()
    want = oracle.check(g.trace(racy))
    assert _races(raw) == [tuple(r) for r in want.races] and flags == 0
    assert (len(raw) > 0) == racy
