"""a9 ring overflow is recovered exactly ("report
races on unique memory addresses"): with a ring far too small, every kernel's
dropped global records come back from the end-of-kernel shadow scan and every
block's dropped shared records from its end-of-block instance spill, so the
report still equals the oracle's racy set — for every replay kernel, across
many kernels, under lazy reset / double shadow / SMEM32, through the async
report, and for online-instrumented kernels.  A spill that is itself too
small must make the report fail (HR_E_INCOMPLETE), never return a short set.
"""
import random

import numpy as np
import pytest

import oracle
from tests.helpers import filter_trace_words
from tests.test_gpu_parity import _concat, _random_batch, gpu_set, oracle_set
from tracegen import c4, stencil
from tracegen import format as tf
from tracegen import programs as tp

pytestmark = pytest.mark.gpu


def hr():
    from paper_2401_04701_b200 import hirace
    return hirace


# kernel choices: row (64 regs), row (32 regs), pooled, pooled-wide (compacted), block-serial,
# run-time options (SMEM32), lazy reset, double shadow
KERNELS = [16, 65536, 32, 256, 32 | 16384, 4096, 8192, 64]


def _multi_kernel_trace():
    """Five kernels, each with far more racy words than a ring of 8 holds, in
    both spaces (global listing-2 style and shared random programs)."""
    rng = random.Random(5)                 # seed: every kernel has > 8 racy words (checked below)
    parts = [tp.listing2(4, 4, 32), tp.listing2(3, 8, 32)]
    for _ in range(3):
        parts.append(tp.random_program(rng, max_blocks=6, max_warps=4, max_lanes=32, max_slots=14,
                                       n_words=300, spaces=(0, 1), p_barrier=0.15, p_skip=0.3))
    return _concat(parts)


@pytest.mark.parametrize("options", KERNELS)
def test_every_kernel_overflows_multi_kernel(options):
    tr = _multi_kernel_trace()
    want, _ = oracle_set(tr)
    per_kernel = {k: sum(1 for r in want if r[0] == k) for k in range(5)}
    assert all(n > 8 for n in per_kernel.values()), per_kernel
    assert any(r[1] == 1 for r in want) and any(r[1] == 0 for r in want)
    g, fl = gpu_set(tr, ring_capacity=8, options=options)
    assert fl & hr().HR_F_RING_OVERFLOW and not fl & hr().HR_F_INCOMPLETE
    assert g == want


@pytest.mark.parametrize("options", [0, 65536, 4096, 32 | 16384])
def test_c3_stencil_shared_overflow(options):
    """C3 (shared-memory stencil, n=128: 64 blocks x 256 threads, one inter-sweep
    barrier removed) with a ring of 8: the racy shared words of every block
    come back through the end-of-block spill."""
    tr = stencil.stencil_trace(removed=20, n=128)
    want, _ = oracle_set(tr)
    assert len(want) > 1000 and all(r[1] == 1 for r in want)
    g, fl = gpu_set(tr, ring_capacity=8, options=options)
    assert fl & hr().HR_F_RING_OVERFLOW
    assert g == want


def test_overflow_random_programs_all_kernels():
    for seed in range(3):
        tr = _random_batch(100 + seed, 6, max_blocks=5, max_warps=6, max_lanes=32, max_slots=10, n_words=60,
                           spaces=(0, 1), p_barrier=0.2, p_skip=0.4)
        want, _ = oracle_set(tr)
        for options in KERNELS:
            for cap in (1, 5):
                assert gpu_set(tr, ring_capacity=cap, options=options)[0] == want, (seed, options, cap)


def test_overflow_host_chunked_and_packed(monkeypatch):
    """Host-buffer replay splits a kernel into several launches (block chunks):
    the spill scan still runs once per kernel, after its last chunk."""
    h = hr()
    monkeypatch.setenv("HR_HOST_CHUNK_BYTES", "4096")
    tr = _multi_kernel_trace()
    want, _ = oracle_set(tr)
    gmax, smem = h.trace_extent(tr)
    ck = h.Checker(gmax, smem, ring_capacity=8)
    ck.replay_host(tr)
    races, fl, _ = ck.report()
    assert [tuple(r) for r in races] == want and fl & h.HR_F_RING_OVERFLOW
    ck.reset()
    packed = ck.pack(h.DeviceTrace.from_trace(tr)).to_host()
    ck.replay_host(packed)
    races, fl, _ = ck.report()
    assert [tuple(r) for r in races] == want
    ck.close()


def test_overflow_shards():
    h = hr()
    tr = _multi_kernel_trace()
    want, _ = oracle_set(tr)
    gmax, smem = h.trace_extent(tr)
    for n, g in ((2, 3), (4, 0), (8, 5)):
        union = []
        for r in range(n):
            ck = h.Checker(gmax, smem, shard=(r, n), granule_log2=g, ring_capacity=3)
            ck.replay(h.DeviceTrace.from_trace(tr))
            races, fl, _ = ck.report()
            ck.close()
            union += [tuple(x) for x in races]
        assert sorted(union) == want


def test_overflow_async_report_falls_back_exactly():
    h = hr()
    tr = _multi_kernel_trace()
    want, _ = oracle_set(tr)
    gmax, smem = h.trace_extent(tr)
    ck = h.Checker(gmax, smem, ring_capacity=8)
    dt = h.DeviceTrace.from_trace(tr)
    for _ in range(2):
        ck.reset()
        ck.replay(dt)
        ck.report_async()
        raw, fl = ck.collect_raw()
        assert h.races_of(raw) == [h.Race(*r) for r in want] and fl & h.HR_F_RING_OVERFLOW
    ck.close()


def test_spill_too_small_fails_loudly():
    h = hr()
    tr = tp.listing2(4, 8, 32)
    gmax, smem = h.trace_extent(tr)
    ck = h.Checker(gmax, smem, ring_capacity=8, spill_capacity=4)
    ck.replay(h.DeviceTrace.from_trace(tr))
    with pytest.raises(h.HiraceError) as e:
        ck.report()
    assert e.value.status == h.HR_E_INCOMPLETE
    ck.report_async()
    with pytest.raises(h.HiraceError) as e:
        ck.collect_raw()
    assert e.value.status == h.HR_E_INCOMPLETE
    ck.close()
    # shared space: a spill of 2 cannot hold one block's racy instance
    tr = stencil.stencil_trace(removed=20, n=32)
    gmax, smem = h.trace_extent(tr)
    ck = h.Checker(gmax, smem, ring_capacity=8, spill_capacity=2)
    ck.replay(h.DeviceTrace.from_trace(tr))
    with pytest.raises(h.HiraceError) as e:
        ck.report()
    assert e.value.status == h.HR_E_INCOMPLETE
    ck.close()


def test_c4_lv20_default_ring():
    """C4 at 2^20 vertices with the DEFAULT ring (2^20 records)."""
    g = c4.Graph(20)
    tr = g.trace(True)
    want = oracle.check(tr)
    got, flags = hr().check_trace(tr)
    assert [tuple(r) for r in got] == [tuple(r) for r in want.races]
    assert flags == want.flags == 0 or flags == hr().HR_F_RING_OVERFLOW


def test_c4_lv20_small_ring():
    """Same graph, ring of 2^10: every BFS level overflows."""
    g = c4.Graph(20)
    tr = g.trace(True)
    want = oracle.check(tr)
    got, flags = hr().check_trace(tr, ring_capacity=1 << 10)
    assert flags & hr().HR_F_RING_OVERFLOW
    assert [tuple(r) for r in got] == [tuple(r) for r in want.races]


def test_c4_full_size_default_ring_sampled():
    """C4 at the BASELINE size (2^24 vertices, ~7.4 M racy words over its
    kernels) at the default 2^20-record ring.  Every sampled word's verdict and
    scope equals the oracle's on the sampled words' exact access histories
    (words are independent FSMs), and the whole set equals the one a ring
    large enough never to overflow collects (no spill involved)."""
    h = hr()
    g = c4.Graph(24)
    tr = g.trace(True)
    got, flags = h.check_trace(tr)
    assert flags == h.HR_F_RING_OVERFLOW
    assert len(got) > (1 << 20)
    got_set = {(r.kernel, r.word, r.scope) for r in got}
    rng = random.Random(12)
    sample = set(rng.sample(range(g.n), 3000)) | set(range(64)) | set(range(g.n, g.n + 1024))
    ref = oracle.check(filter_trace_words(tr, sample))
    want = {(r.kernel, r.word, r.scope) for r in ref.races}
    assert {x for x in got_set if x[1] in sample} == want
    assert len(want) > 100
    big, bflags = h.check_trace(tr, ring_capacity=1 << 24)
    assert bflags == 0 and big == got


# ---- online kernels (include/hr_bench.h): hr_thread_end spills shared races ----

def _races(raw):
    return [(int(r["kernel"]), int(r["space"]), int(r["block"]), int(r["word"]), int(r["scope"])) for r in raw]


@pytest.mark.parametrize("options", [0, 4096])
def test_online_c3_overflow(options):
    import torch
    from paper_2401_04701_b200 import online
    h = hr()
    n = 128
    data = torch.randint(0, 100, (2 * n * n,), dtype=torch.int32, device="cuda")
    ck = h.Checker(2 * n * n, 648, ring_capacity=8, options=options)
    online.c3(ck.ctx, data, True, n=n, removed=20)
    raw, flags = ck.report_raw()
    want = oracle.check(stencil.stencil_trace(removed=20, n=n))
    assert _races(raw) == [tuple(r) for r in want.races] and flags == h.HR_F_RING_OVERFLOW


def test_online_c1_wrapper_overflow():
    import torch
    from paper_2401_04701_b200 import online
    h = hr()
    data = torch.arange(8 * 256 + 8, dtype=torch.int32, device="cuda")
    ck = h.Checker(8 * 256 + 8, 256, ring_capacity=2)
    online.c1_array(ck.ctx, data, removed=32)
    raw, flags = ck.report_raw()
    want = oracle.check(tp.c1_tree_reduction(removed=32))
    assert _races(raw) == [tuple(r) for r in want.races] and flags == h.HR_F_RING_OVERFLOW


def test_online_c4_overflow_and_async():
    """Online C4 (one kernel id per BFS level + the histogram) with a small
    ring: global drops of every level are scanned; the async report over
    online kernel ids (any id) equals the sync one."""
    import torch
    from paper_2401_04701_b200 import online
    h = hr()
    g = c4.Graph(16)
    dev = online.C4Device(g)
    want = [tuple(r) for r in oracle.check(g.trace(True)).races]
    for ring in (1 << 4, 1 << 20):
        data = torch.full((g.n + 1024,), -1, dtype=torch.int32, device="cuda")
        data[g.n:] = 0
        ck = h.Checker(g.n + 1024, 0, ring_capacity=ring)
        dev.run(ck.ctx, data, True, True)
        raw, _ = ck.report_raw()
        assert _races(raw) == want
        ck.reset()
        data[: g.n] = -1
        data[g.n:] = 0
        dev.run(ck.ctx, data, True, True, kernel_base=1000)
        ck.report_async()
        a_raw, _ = ck.collect_raw()
        s_raw, _ = ck.report_raw()
        assert _races(a_raw) == _races(s_raw) == [(r[0] + 1000,) + r[1:] for r in want]
        ck.close()


@pytest.mark.parametrize("options", [8192, 64])
def test_online_after_replay_same_ctx(options):
    """Replay, then online kernels on the same ctx under lazy reset / double
    shadow: the online kernel must see a fresh shadow epoch (hr_kernel_begin
    before hr_device_view), so no false cross-kernel races."""
    import torch
    from paper_2401_04701_b200 import online
    h = hr()
    g = c4.Graph(14)
    dev = online.C4Device(g)
    tr = g.trace(False)                         # race-free atomic variant: touches the same words
    ck = h.Checker(g.n + 1024, 0, options=options)
    ck.replay(h.DeviceTrace.from_trace(tr))
    data = torch.full((g.n + 1024,), -1, dtype=torch.int32, device="cuda")
    data[g.n:] = 0
    for _ in range(3):
        dev.run(ck.ctx, data, True, False, kernel_base=50)
    raw, flags = ck.report_raw()
    assert len(raw) == 0 and flags == 0
    ck.close()


def test_async_then_large_sync_then_async():
    """an hr_report_async, then a large synchronous report
    (device sort that regrows the pinned staging), then async again on the
    same ctx."""
    h = hr()
    small = tp.listing2(2, 2, 32)
    big = tp.listing2(64, 8, 32)                     # > 4096 races
    gmax, smem = h.trace_extent(big)
    ck = h.Checker(gmax, smem)
    for tr in (small, big, small, big):
        want, _ = oracle_set(tr)
        dt = h.DeviceTrace.from_trace(tr)
        ck.reset(); ck.replay(dt); ck.report_async()
        a_raw, _ = ck.collect_raw()
        ck.reset(); ck.replay(dt)
        s_raw, _ = ck.report_raw()
        assert _races(a_raw) == _races(s_raw) == want
    ck.close()
