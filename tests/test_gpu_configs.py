"""GPU parity on the BASELINE.json configs, through the C ABI.

C2: all ~588 suite traces, element by element vs the oracle.
C3: the full 1024-block stencil (2^26 accesses), racy and race-free, vs the oracle.
C5: GPU generator == CPU generator bit for bit; small C5 vs the oracle; the
    full 2^32-access trace (the configuration bench.py times) vs its closed
    form (the planted set — exact by construction, pinned by the oracle at
    small sizes in tests/test_configs.py).
"""
import numpy as np
import pytest

import oracle
from tracegen import c5, stencil, suite

pytestmark = pytest.mark.gpu


def hr():
    from paper_2401_04701_b200 import hirace
    return hirace


def test_c2_suite_parity():
    h = hr()
    cases = suite.suite()
    racy = 0
    for c in cases:
        got, flags = h.check_trace(c.trace)
        want = oracle.check(c.trace)
        assert [tuple(r) for r in got] == [tuple(r) for r in want.races], c.name
        assert flags == want.flags == 0, c.name
        racy += bool(got)
    assert racy == sum(c.racy for c in cases)


@pytest.mark.parametrize("removed", [20, None])
def test_c3_full_size_parity(removed):
    tr = stencil.stencil_trace(removed=removed)
    got, flags = hr().check_trace(tr)
    want = oracle.check(tr)
    assert flags == want.flags == 0
    assert [tuple(r) for r in got] == [tuple(r) for r in want.races]
    assert len(got) == (1024 * 512 if removed is not None else 0)


@pytest.mark.parametrize("nshard", [1, 2, 8])
def test_c5_gpu_generator_matches_cpu(nshard):
    import torch
    lb = 3
    for rank in range(nshard):
        cpu = c5.cpu_trace(lb, rank=rank, nshard=nshard)
        rec, off, kd = c5.gpu_trace(lb, rank=rank, nshard=nshard)
        assert np.array_equal(off.cpu().numpy().view(np.uint64), cpu.warp_off)
        assert np.array_equal(rec.cpu().numpy().view(np.uint64), cpu.rec)
        assert np.array_equal(kd, cpu.kdesc)


def test_c5_small_vs_oracle():
    tr = c5.cpu_trace(6)
    got, flags = hr().check_trace(tr)
    want = oracle.check(tr)
    assert [tuple(r) for r in got] == [tuple(r) for r in want.races] and flags == 0


def test_c5_full_size_closed_form():
    """The bench configuration: 2^16 blocks, 2^32 accesses, 2^32-word shadow."""
    import torch
    h = hr()
    lb = 16
    rec, off, kd = c5.gpu_trace(lb)
    ck = h.Checker(c5.total_words(lb), 0, ring_capacity=1 << 20)
    ck.replay(h.DeviceTrace(rec, off, kd))
    raw, flags = ck.report_raw()
    ck.close()
    del rec
    torch.cuda.empty_cache()
    assert flags == 0
    assert [(int(r["word"]), int(r["scope"])) for r in raw] == c5.planted(lb)
    assert all(int(r["kernel"]) == 0 and int(r["space"]) == 0 and int(r["block"]) == 0xFFFFFFFF for r in raw)


@pytest.mark.parametrize("nshard", [1, 4])
def test_c5_gpu_compact_generator_matches_cpu(nshard):
    from tracegen.format import to_c32
    lb = 3
    for rank in range(nshard):
        cpu = c5.cpu_trace(lb, rank=rank, nshard=nshard)
        r32, rop = to_c32(cpu)
        g32, grop, off, kd = c5.gpu_trace_c32(lb, rank=rank, nshard=nshard)
        assert np.array_equal(g32.cpu().numpy().view(np.uint32), r32)
        assert np.array_equal(grop.cpu().numpy(), rop)
        assert np.array_equal(off.cpu().numpy().view(np.uint64), cpu.warp_off)


def test_c5_full_size_compact_closed_form():
    import torch
    h = hr()
    lb = 16
    r32, rop, off, kd = c5.gpu_trace_c32(lb)
    ck = h.Checker(c5.total_words(lb), 0, ring_capacity=1 << 20)
    ck.replay(h.DeviceTrace(None, off, kd, r32, rop))
    raw, flags = ck.report_raw()
    ck.close()
    del r32, rop
    torch.cuda.empty_cache()
    assert flags == 0
    assert [(int(r["word"]), int(r["scope"])) for r in raw] == c5.planted(lb)
