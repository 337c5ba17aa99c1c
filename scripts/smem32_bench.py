"""HR_OPT_SMEM32 vs the 64-bit shared shadow: replay kernel time of the
shared-shadow configs (C1, C3) and the online C3 kernel.  Not the driver's
bench; a measurement tool for DESIGN.md §9."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2401_04701_b200 import hirace as hr, online as on  # noqa: E402
from tracegen import programs, stencil  # noqa: E402


def replay_ms(tr, opts, reps=10):
    dt = hr.DeviceTrace.from_trace(tr)
    gmax, smem = hr.trace_extent(tr)
    ck = hr.Checker(gmax, smem, options=hr.HR_OPT_TIMING | opts)
    for _ in range(3):
        ck.reset(); ck.replay(dt); ck.report_raw()
    hr.hr_replay_timing(ck.ctx)
    for _ in range(reps):
        ck.reset(); ck.replay(dt); raw, fl = ck.report_raw()
    _, _, kms, nk = hr.hr_replay_timing(ck.ctx)
    ck.close()
    return kms / nk, len(raw), fl


out = {}
for name, tr in (("c1", programs.c1_tree_reduction(removed=32)), ("c3", stencil.stencil_trace(removed=20))):
    for label, o in (("smem64", 0), ("smem32", hr.HR_OPT_SMEM32)):
        ms, n, fl = replay_ms(tr, o)
        out[f"{name}_{label}"] = {"kernel_ms": round(ms, 4), "races": n, "flags": fl,
                                  "smem_shadow_bytes_per_block": hr.trace_extent(tr)[1] * (4 if o else 8)}
d3 = torch.randint(0, 100, (2 * 512 * 512,), dtype=torch.int32, device="cuda")
for label, o in (("smem64", 0), ("smem32", hr.HR_OPT_SMEM32)):
    ck = hr.Checker(2 * 512 * 512, 648, options=o)
    out[f"c3_online_{label}"] = on.slowdown(lambda: on.c3(None, d3, False), lambda: on.c3(ck.ctx, d3, True), reps=10)
    ck.close()
print(json.dumps(out))
