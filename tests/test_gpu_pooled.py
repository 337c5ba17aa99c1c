"""HR_TRACE_POOLED (include/hr.h, hr_pool_trace): the same access streams laid
out as warp pools — up to 32 accesses of one simulated warp inside one
epoch per row, with their simulated lanes as tags.  Replaying the pooled
layout must give exactly the oracle's racy set and flags; on an address
shard the pooling drops the records the rank does not own (the per-rank
input of the multi-GPU replay)."""
import random

import numpy as np
import pytest

from tests.test_gpu_parity import _concat, _only_representatives, _random_batch, gpu_set, oracle_set
from tracegen import c5, stencil
from tracegen import programs as tp

pytestmark = pytest.mark.gpu


def hr():
    from paper_2401_04701_b200 import hirace
    return hirace


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("options", [0, 4096, 8192, 1 | 2])
def test_pooled_random_programs(seed, options):
    tr = _random_batch(900 + seed, 20, max_blocks=6, max_warps=8, max_lanes=32, max_slots=14, n_words=50,
                       spaces=(0, 1), p_barrier=0.25, p_skip=0.6)
    want = oracle_set(tr)
    assert gpu_set(tr, pooled=True, options=options) == want
    assert gpu_set(tr, pooled=True, compact=True, options=options) == want


def test_pooled_listings_c1_c3_suite():
    from tracegen import suite
    cases = [tp.listing1(2, 2, 32), tp.listing2(4, 4, 32), tp.listing4(1, 2, 32, 40),
             tp.c1_tree_reduction(removed=16), stencil.stencil_trace(removed=20, n=64)]
    cases += [c.trace for c in suite.suite()[::9]]
    for tr in cases:
        assert gpu_set(tr, pooled=True) == oracle_set(tr)


def test_pooled_representatives():
    tr = _random_batch(77, 10, max_blocks=6, max_warps=8, max_lanes=32, max_slots=12, n_words=40,
                       spaces=(0, 1), p_barrier=0.25, p_skip=0.5)
    for reps in ((2, 1), (1, 2)):
        assert gpu_set(tr, pooled=True, representatives=reps) == oracle_set(_only_representatives(tr, *reps))


def test_pooled_shards_union_and_c5_planted():
    h = hr()
    tr = _random_batch(31, 12, max_blocks=4, max_warps=8, max_lanes=32, max_slots=10, n_words=3000,
                       spaces=(0, 1))
    want, _ = oracle_set(tr)
    gmax, smem = h.trace_extent(tr)
    for n in (2, 8):
        union = []
        for r in range(n):
            ck = h.Checker(gmax, smem, shard=(r, n))
            ck.replay(ck.pool(h.DeviceTrace.from_trace(tr)))
            union += [tuple(x) for x in ck.report()[0]]
            ck.close()
        assert sorted(union) == want
    # C5 shard traces (the bench's per-rank input), pooled from C32
    lb, n = 8, 8
    union = []
    for r in range(n):
        r32, rop, woff, kd = c5.gpu_trace_c32(lb, rank=r, nshard=n)
        ck = h.Checker(c5.total_words(lb), 0, shard=(r, n), options=h.HR_OPT_LAZY_RESET)
        dt = h.DeviceTrace(None, woff, kd, r32, rop)
        pooled = ck.pool(dt)
        assert pooled.n_rows < dt.n_rows
        for _ in range(2):
            ck.reset()
            ck.replay(pooled)
            raw, fl = ck.report_raw()
        assert fl == 0
        union += [(int(x["word"]), int(x["scope"])) for x in raw]
        ck.close()
    assert sorted(union) == c5.planted(lb)


@pytest.mark.parametrize("options", [0, 16, 32, 256, 16384 | 32])
def test_shard_owned_flag_same_result(options):
    """HR_TRACE_F_SHARD_OWNED (the per-access owner hash skipped for traces
    partitioned for this rank): same per-rank sets as the owner test, on C5
    shards from the generator and on host-sharded random programs."""
    from paper_2401_04701_b200 import multigpu
    h = hr()
    lb, n = 8, 8
    union = []
    for r in range(n):
        r32, rop, woff, kd = c5.gpu_trace_c32(lb, rank=r, nshard=n)
        ck = h.Checker(c5.total_words(lb), 0, shard=(r, n), options=options | h.HR_OPT_LAZY_RESET)
        dt = h.DeviceTrace(None, woff, kd, r32, rop)
        ck.replay(dt)
        plain = [tuple(x) for x in ck.report()[0]]
        ck.reset()
        dt.flags = h.HR_TRACE_F_SHARD_OWNED
        ck.replay(dt)
        owned = [tuple(x) for x in ck.report()[0]]
        ck.close()
        assert owned == plain
        union += owned
    assert sorted((x[3], x[4]) for x in union) == c5.planted(lb)
    tr = _random_batch(61, 8, max_blocks=4, max_warps=8, max_lanes=32, max_slots=10, n_words=3000, spaces=(0, 1))
    want, _ = oracle_set(tr)
    gmax, smem = h.trace_extent(tr)
    union = []
    for r in range(4):
        ck = h.Checker(gmax, smem, shard=(r, 4), options=options)
        dt = h.DeviceTrace.from_trace(multigpu.shard_trace(tr, r, 4))
        dt.flags = h.HR_TRACE_F_SHARD_OWNED
        ck.replay(dt)
        union += [tuple(x) for x in ck.report()[0]]
        ck.close()
    assert sorted(union) == want
