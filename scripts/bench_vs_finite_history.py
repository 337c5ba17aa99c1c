"""HiRace vs the finite-history baseline (HR_OPT_FINITE_HISTORY: iGUARD-style
one-reader/one-writer 16-byte records) on the same replay.

Reproduces the paper's comparisons on this box, with our own baseline in
place of iGUARD (which does not run here):
  * completeness: Listing 4's eviction omission and the
    C2 suite's racy traces found / missed (the shape of Table II);
  * memory: 8 vs 16 bytes per monitored word;
  * speed: kernel time on C3 (SMEM shadow) and C5 (HBM, hot atomic words;
    the paper: ">10x faster than iGUARD").
Writes profiles/r01_vs_finite_history.json.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import oracle  # noqa: E402  (test infrastructure: ground truth for the completeness counts)
from paper_2401_04701_b200 import hirace as hr  # noqa: E402
from tracegen import c5, programs as tp, stencil, suite  # noqa: E402

FH = hr.HR_OPT_FINITE_HISTORY


def time_kernel(dt, words, smem, opt, reps=3):
    ck = hr.Checker(words, smem, options=hr.HR_OPT_TIMING | opt, ring_capacity=1 << 22)
    for _ in range(1):
        ck.reset(); ck.replay(dt); ck.report_raw()
    hr.hr_replay_timing(ck.ctx)
    for _ in range(reps):
        ck.reset(); ck.replay(dt); raw, fl = ck.report_raw()
    r = hr.hr_replay_timing(ck.ctx)
    ck.close()
    return r[2] / reps, len(raw)


def main():
    out = {}
    # completeness
    tr = tp.listing4(1, 1, 4, 4)
    out["listing4_1x1x4"] = {"oracle": len(oracle.check(tr).races),
                             "hirace": len(hr.check_trace(tr)[0]),
                             "finite_history": len(hr.check_trace(tr, options=FH)[0])}
    racy = found_h = found_f = words_total = words_h = words_f = 0
    for c in suite.suite():
        want = {(r.kernel, r.space, r.block, r.word) for r in oracle.check(c.trace).races}
        gh = {tuple(r[:4]) for r in hr.check_trace(c.trace)[0]}
        gf = {tuple(r[:4]) for r in hr.check_trace(c.trace, options=FH)[0]}
        assert gh == want and gf <= want
        if want:
            racy += 1
            found_h += bool(gh)
            found_f += bool(gf)
            words_total += len(want)
            words_h += len(gh)
            words_f += len(gf)
    out["c2_suite"] = {"racy_traces": racy, "hirace_found": found_h, "finite_history_found": found_f,
                       "racy_words": words_total, "hirace_words": words_h, "finite_history_words": words_f}
    out["bytes_per_word"] = {"hirace": 8, "finite_history": 16}
    # speed
    dt3 = hr.DeviceTrace.from_trace(stencil.stencil_trace(removed=20))
    h3, n3 = time_kernel(dt3, 2 * 512 * 512, 648, 0)
    f3, m3 = time_kernel(dt3, 2 * 512 * 512, 648, FH)
    out["c3_kernel_ms"] = {"hirace": h3, "finite_history": f3, "races": [n3, m3]}
    del dt3
    lb = 12
    dt5 = hr.DeviceTrace(*c5.gpu_trace(lb))
    h5, n5 = time_kernel(dt5, c5.total_words(lb), 0, 0)
    f5, m5 = time_kernel(dt5, c5.total_words(lb), 0, FH, reps=1)
    out[f"c5_2^{lb + 16}_kernel_ms"] = {"hirace": h5, "finite_history": f5, "speedup": f5 / h5, "races": [n5, m5]}
    print(json.dumps(out, indent=1))
    with open(os.path.join(ROOT, "profiles", "r01_vs_finite_history.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
