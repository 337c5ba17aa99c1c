"""Where the non-kernel part of a C5 bench step goes (diagnostic)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_04701_b200 import hirace as hr
from tracegen import c5
lb = int(sys.argv[1]) if len(sys.argv) > 1 else 16
rec, woff, kd = c5.gpu_trace(lb)
dt = hr.DeviceTrace(rec, woff, kd)
ck = hr.Checker(c5.total_words(lb), 0, ring_capacity=1 << 21, options=hr.HR_OPT_TIMING)
s = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    ck.reset(); ck.replay(dt, s); ck.report_raw()
hr.hr_replay_timing(ck.ctx)
for _ in range(int(os.environ.get("STEPS", "3"))):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    ck.reset(); torch.cuda.synchronize(); t1 = time.perf_counter()
    ck.replay(dt, s); t2 = time.perf_counter(); torch.cuda.synchronize(); t3 = time.perf_counter()
    raw, fl = ck.report_raw(); t4 = time.perf_counter()
    print(f"reset {1e3*(t1-t0):.2f}  replay-issue {1e3*(t2-t1):.2f}  replay-wait {1e3*(t3-t2):.2f}  report {1e3*(t4-t3):.2f} ms  races {len(raw)}")
print("device timing", hr.hr_replay_timing(ck.ctx))
import ctypes, numpy as np
lib = hr.load()
for cap in (1 << 17, 1 << 20):
    buf = np.empty(cap, dtype=hr.RACE_DTYPE)
    n = ctypes.c_size_t(0); fl = ctypes.c_uint32(0)
    ck.reset(); ck.replay(dt, s); torch.cuda.synchronize()
    t0 = time.perf_counter()
    rc = lib.hr_report(ck.ctx, buf.ctypes.data_as(ctypes.POINTER(hr.HrRace)), cap, ctypes.byref(n), ctypes.byref(fl))
    t1 = time.perf_counter()
    print(f"C hr_report cap {cap}: {1e3*(t1-t0):.2f} ms rc {rc} n {n.value}")
