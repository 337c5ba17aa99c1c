"""Profiling driver for one replay config (ncu target).  Not a bench."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_04701_b200 import hirace as hr
from tracegen import c4, stencil

ap = argparse.ArgumentParser()
ap.add_argument("config", choices=["c3", "c4"])
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--lv", type=int, default=20, help="C4 graph: 2^lv vertices")
ap.add_argument("--atomic", action="store_true", help="C4 race-free (atomic) variant")
ap.add_argument("--u64", action="store_true", help="U64 records (default: C32, as bench.py)")
ap.add_argument("--racefree", action="store_true", help="C3 race-free variant")
ap.add_argument("--options", type=int, default=0)
ap.add_argument("--online", action="store_true", help="C3: the instrumented online kernel instead of a replay")
a = ap.parse_args()
if a.online:
    import torch
    from paper_2401_04701_b200 import online as on
    d3 = torch.zeros(2 * 512 * 512, dtype=torch.int32, device="cuda")
    ck = hr.Checker(2 * 512 * 512, 648, ring_capacity=1 << 24, options=a.options)
    for _ in range(a.reps):
        ck.reset(); on.c3(ck.ctx, d3, True, removed=None if a.racefree else 20); raw, fl = ck.report_raw()
    print("races", len(raw), "flags", fl)
    sys.exit(0)
if a.config == "c3":
    tr, words, smem = stencil.stencil_trace(removed=None if a.racefree else 20), 2 * 512 * 512, 648
else:
    g = c4.Graph(a.lv)
    tr, words, smem = g.trace(not a.atomic), c4.total_words(a.lv), 0
dt = hr.DeviceTrace.from_trace(tr, compact=not a.u64)
ck = hr.Checker(words, smem, ring_capacity=1 << 24, options=hr.HR_OPT_TIMING | a.options)
for _ in range(a.reps):
    ck.reset(); ck.replay(dt); raw, fl = ck.report_raw()
print("races", len(raw), "flags", fl, hr.hr_replay_timing(ck.ctx))
