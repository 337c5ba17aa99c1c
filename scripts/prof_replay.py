"""Profiling driver: generate C5 at 2^lb blocks in HBM and replay it `reps` times
(so ncu can capture a warm launch).  Not a bench: numbers printed here under a
profiler are never reported."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_04701_b200 import hirace as hr
from tracegen import c5

ap = argparse.ArgumentParser()
ap.add_argument("--lb", type=int, default=12)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--options", type=int, default=0)
ap.add_argument("--format", default="c32", choices=["c32", "u64"])
ap.add_argument("--shard", default="0/1", help="R/N: replay address shard R of N")
ap.add_argument("--granule", type=int, default=9, help="log2 words of an address-shard granule")
a = ap.parse_args()
sr, sn = (int(x) for x in a.shard.split("/"))
if a.format == "c32":
    r32, rop, woff, kd = c5.gpu_trace_c32(a.lb, rank=sr, nshard=sn, granule_log2=a.granule)
    dt = hr.DeviceTrace(None, woff, kd, r32, rop)
else:
    rec, woff, kd = c5.gpu_trace(a.lb, rank=sr, nshard=sn, granule_log2=a.granule)
    dt = hr.DeviceTrace(rec, woff, kd)
ck = hr.Checker(c5.total_words(a.lb), 0, options=a.options | hr.HR_OPT_TIMING, ring_capacity=1 << 21, shard=(sr, sn),
                granule_log2=a.granule)
for i in range(a.reps):
    ck.reset(); ck.replay(dt); raw, fl = ck.report_raw()
print("races", len(raw), "flags", fl, "timing", hr.hr_replay_timing(ck.ctx))
