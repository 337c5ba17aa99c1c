"""Device counters of the check (diagnostic build): checked accesses, failed
CAS (Algorithm 1 retries), a7 fast exits, committed CAS per config.  Run with
HIRACE_LIB pointing at a -DHR_COUNTERS build (the production build keeps no
counters).  Not a bench: the counting atomics slow the replay down."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2401_04701_b200 import hirace as hr  # noqa: E402
from tracegen import c4, c5, stencil  # noqa: E402


def run(name, dt, words, smem=0, ring=1 << 22, opts=0):
    ck = hr.Checker(words, smem, ring_capacity=ring, options=opts)
    ck.reset()
    ck.replay(dt)
    raw, fl = ck.report_raw()
    n = hr.hr_counters(ck.ctx)
    ck.close()
    out = {"config": name, "checked": n[0], "cas_failed_retries": n[1], "fast_exits": n[2], "cas_committed": n[3],
           "races": len(raw), "flags": fl}
    if n[0]:
        out.update({"retries_per_check": n[1] / n[0], "fast_exit_share": n[2] / n[0],
                    "cas_per_check": (n[1] + n[3]) / n[0]})
    print(json.dumps(out), flush=True)
    return out


if __name__ == "__main__":
    lb = int(os.environ.get("C5_LB", "16"))
    r32, rop, woff, kd = c5.gpu_trace_c32(lb)
    run(f"C5 2^{lb + 16} accesses", hr.DeviceTrace(None, woff, kd, r32, rop), c5.total_words(lb), opts=hr.HR_OPT_LAZY_RESET)
    del r32, rop
    torch.cuda.empty_cache()
    run("C3 stencil race-free", hr.DeviceTrace.from_trace(stencil.stencil_trace(removed=None), compact=True),
        2 * 512 * 512, 648)
    run("C3 stencil racy", hr.DeviceTrace.from_trace(stencil.stencil_trace(removed=20), compact=True), 2 * 512 * 512, 648)
    g = c4.Graph(24)
    for racy in (True, False):
        run(f"C4 2^24 {'racy' if racy else 'atomic'}", hr.DeviceTrace.from_trace(g.trace(racy), compact=True),
            c4.total_words(24), ring=1 << 24)
