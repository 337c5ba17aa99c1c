"""Micro-benchmark of one long sparse warp (the C4 level-0 hub shape): one
block, one warp, lane 0 issues R w; W w for n random words over 2^24, the other
31 lanes are NOP.  Times the replay kernel alone (not a bench)."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2401_04701_b200 import hirace as hr
from tracegen import format as tf

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=369000)
ap.add_argument("--options", type=int, default=hr.HR_OPT_POOL_WIDE)
ap.add_argument("--lanes", type=int, default=1, help="active lanes per row")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
rng = np.random.default_rng(1)
W = 1 << 24
words = rng.integers(0, W, (a.n, a.lanes)).astype(np.uint64)
rows = np.full((2 * a.n, 32), tf.NOP, dtype=np.uint64)
rows[0::2, :a.lanes] = words                                   # R
rows[1::2, :a.lanes] = (np.uint64(1) << np.uint64(62)) | words   # W
tr = tf.Trace(rows.reshape(-1), np.array([[1, 1, 32, 0, 0, 0, 0, 0]], dtype=np.uint64),
              np.array([0, 2 * a.n], dtype=np.uint64))
dt = hr.DeviceTrace.from_trace(tr)
ck = hr.Checker(W, 0, options=a.options | hr.HR_OPT_TIMING, ring_capacity=1 << 22)
for _ in range(a.reps):
    ck.reset(); ck.replay(dt); raw, fl = ck.report_raw()
_, _, kms, nk = hr.hr_replay_timing(ck.ctx)
print(f"rows {2 * a.n} lanes {a.lanes} kernel {kms / nk:.3f} ms  {1e6 * kms / nk / (2 * a.n):.1f} ns/row  races {len(raw)}")
