"""Replay throughput of every BASELINE config on one GPU (checked accesses/s,
kernel ms from HR_OPT_TIMING events).  Not the driver's bench (bench.py);
a per-config measurement tool.  Usage: python scripts/bench_configs.py [c1 c2 c3 c4 c5]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2401_04701_b200 import hirace as hr  # noqa: E402
from tracegen import c4, c5, programs, stencil, suite  # noqa: E402


def raw_ms(dt, words, reps=3):
    """The uninstrumented replay of the same records (hrb_raw_replay)."""
    from paper_2401_04701_b200 import online as on
    data = torch.zeros(words, dtype=torch.int32, device="cuda")
    t = on.time_ms(lambda: on.raw_replay(dt, data, words), reps=reps, warmup=1)
    del data
    return t


def run(name, trace=None, dt=None, words=None, smem=0, reps=5, ring=1 << 22, opts=0):
    if dt is None:
        dt = hr.DeviceTrace.from_trace(trace)
    n_acc = int(((dt.rec >> 62) & 3).ne(3).sum().item())
    opts |= int(os.environ.get("HR_OPTS", "0"))
    ck = hr.Checker(words, smem, ring_capacity=ring, options=hr.HR_OPT_TIMING | opts)
    for _ in range(2):
        ck.reset(); ck.replay(dt); ck.report_raw()
    hr.hr_replay_timing(ck.ctx)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        ck.reset(); ck.replay(dt); raw, fl = ck.report_raw()
    wall = (time.perf_counter() - t0) / reps
    rms, nr, kms, nk = hr.hr_replay_timing(ck.ctx)
    kms /= reps
    ck.close()
    rms_raw = raw_ms(dt, words) if os.environ.get("RAW") else None
    out = {"config": name, "accesses": n_acc, "kernels": nk // reps, "kernel_ms": round(kms, 4),
           "raw_replay_ms": rms_raw, "slowdown_vs_raw": (kms / rms_raw) if rms_raw else None,
           "reset_ms": round(rms / reps, 4), "wall_ms": round(wall * 1e3, 3),
           "kernel_acc_per_s": n_acc / (kms / 1e3), "races": len(raw), "flags": fl}
    print(json.dumps(out), flush=True)
    return out


def main(which):
    if "c1" in which:
        run("C1 tree reduction (removed=32)", programs.c1_tree_reduction(removed=32), words=2056, smem=256, reps=20)
    if "c2" in which:
        cases = suite.suite()
        from tracegen.format import make_trace
        # all 588 traces' kernels concatenated into one multi-kernel trace
        ks = []
        for c in cases:
            t = c.trace
            for k in range(t.kdesc.shape[0]):
                b, w, l, sm, woi = (int(x) for x in t.kdesc[k, :5])
                from tracegen.format import Kernel
                kk = Kernel(b, w, l, sm)
                kk.rows = [t.rec[int(t.warp_off[woi + i]) * 32: int(t.warp_off[woi + i + 1]) * 32].reshape(-1, 32)
                           for i in range(b * w)]
                ks.append(kk)
        big = make_trace(ks)
        gmax, smem = hr.trace_extent(big)
        run(f"C2 suite ({len(cases)} traces, {len(ks)} kernels)", big, words=gmax, smem=smem, reps=3)
    if "c3" in which:
        run("C3 stencil racy (removed=20)", stencil.stencil_trace(removed=20), words=2 * 512 * 512, smem=648)
        run("C3 stencil race-free", stencil.stencil_trace(removed=None), words=2 * 512 * 512, smem=648)
    if "c4" in which:
        g = c4.Graph(24)
        for racy in (True, False):
            run(f"C4 BFS+hist 2^24 {'racy' if racy else 'atomic'}", g.trace(racy), words=c4.total_words(24),
                reps=3, ring=1 << 24)
    if "c5" in which:
        rec, off, kd = c5.gpu_trace(16)
        run("C5 2^32", dt=hr.DeviceTrace(rec, off, kd), words=c5.total_words(16), reps=3)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2", "c3", "c4", "c5"])
