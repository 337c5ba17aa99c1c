"""Small replays of every kernel path, for compute-sanitizer (memcheck /
synccheck / racecheck) runs.  Checks results against the oracle too.
--race-free: the online (user) kernels run their race-free variants, so any
racecheck hazard is in the checker itself, not in the program under test."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import oracle
from paper_2401_04701_b200 import hirace as hr, online as on
from tracegen import c4, c5, programs as tp, stencil

def same(tr, **kw):
    got, fl = hr.check_trace(tr, **kw)
    want = oracle.check(tr)
    assert [tuple(r) for r in got] == [tuple(r) for r in want.races] and fl == want.flags, kw

same(tp.c1_tree_reduction(removed=16))
same(stencil.stencil_trace(removed=3, n=32, sweeps=6))
same(tp.listing2(3, 2, 32), options=hr.HR_OPT_POOL)
same(c5.cpu_trace(2), compact=True)
same(c4.Graph(10).trace(True), options=hr.HR_OPT_POOL)
same(tp.listing4(2, 2, 32, 60), options=hr.HR_OPT_DOUBLE_SHADOW)
hr.check_trace(tp.listing4(1, 1, 4, 4), options=hr.HR_OPT_FINITE_HISTORY)
rf = "--race-free" in sys.argv
d = torch.arange(8 * 256 + 8, dtype=torch.int32, device="cuda")
ck = hr.Checker(8 * 256 + 8, 256)
on.c1(ck.ctx, d, True, removed=None if rf else 8); on.c1_array(ck.ctx, d, removed=None if rf else 8)
ck.report_raw(); ck.close()
d3 = torch.zeros(2 * 64 * 64, dtype=torch.int32, device="cuda")
ck = hr.Checker(2 * 64 * 64, 648)
on.c3(ck.ctx, d3, True, n=64, sweeps=6, removed=None if rf else 2); ck.report_raw(); ck.close()
# round 2: the report graph (small-set kernel and the conditional sort path), the
# hybrid binned replay, the PACKED read/write mask, an owned address shard
for tr, n_ring in ((tp.listing2(2, 2, 32), 1 << 12), (tp.listing2(64, 8, 32), 1 << 14)):
    gmax, smem = hr.trace_extent(tr)
    ck = hr.Checker(gmax, smem, ring_capacity=n_ring)
    ck.reset(); ck.replay(hr.DeviceTrace.from_trace(tr)); ck.report_async()
    raw, fl = ck.collect_raw()
    want = oracle.check(tr)
    assert [(int(r["kernel"]), int(r["space"]), int(r["block"]), int(r["word"]), int(r["scope"])) for r in raw] == \
        [tuple(r) for r in want.races]
    ck.close()
same(tp.listing2(4, 4, 32), options=hr.HR_OPT_HYBRID | hr.HR_OPT_BIN_ALL)
same(tp.listing4(2, 2, 32, 60), options=hr.HR_OPT_HYBRID | hr.HR_OPT_BIN_ALL, compact=True)
same(tp.c1_tree_reduction(removed=16), packed=True)
same(c5.cpu_trace(2), packed=True)
torch.cuda.synchronize()
print("sanitize smoke ok")
