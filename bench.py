#!/usr/bin/env python
"""Benchmark: checked accesses/s of the HiRace per-access race check on B200.

Workload (BASELINE.json configs[4], the multi-GPU config the metric is
quoted on): C5 — a 2^32-access global trace over a 2^32-word (16 GiB)
address space, 2^16 blocks x 256 threads x 256 accesses, address-sharded
across N GPUs (tracegen/c5gen.h).  One STEP = one pass of the whole hot path
over the trace: report-ring reset, kernel-boundary reset (a11: epoch tags, a
real memset every 15 kernels), the replay kernel (a1-a10, a12), the report
(a13: at N = 1 hr_report_async, sorted and merged on the device and written
to pinned host memory; at N > 1 hr_report plus the NCCL allgather of the
per-shard race sets).

  value  device-resident: trace generated in HBM before timing; K steps timed
         with CUDA events on the launching stream, max over ranks.
  e2e    same steps through hr_replay_trace_host: the trace lives in pinned
         host memory (HR_TRACE_PACKED by default, decoded on the device) and is
         copied H2D inside every timed step; the race set is read back D2H.
  roofline  for the replay kernel: algorithmic bytes / live event-timed
         duration vs MEASURED_PEAKS.json hbm_gbs.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "checked_accesses_per_sec"
UNIT = "accesses/s"
BYTES_PER_ACCESS_ALGO = 16          # 8 B shadow read + 8 B shadow write-back (a4 + a8)
BYTES_PER_ACCESS_LITERAL = 8        # north_star: "8 B of shadow read-modify-write per checked access"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5", choices=["c5", "c3"],
                    help="c5 (default): the BASELINE metric's workload; c3: the shared-memory stencil "
                         "(BASELINE configs[2]), bound by instruction issue, not HBM")
    ap.add_argument("--lb", type=int, default=16, help="log2 blocks of C5 (16 = full 2^32 accesses)")
    ap.add_argument("--seed", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-lb", type=int, default=10, help="C5 sample for the oracle cpu_baseline")
    ap.add_argument("--ref-lb", type=int, default=8, help="C5 sample per --impl reference step")
    ap.add_argument("--options", type=int, default=0, help="extra HR_OPT_* bits (ablations)")
    ap.add_argument("--no-slowdown", action="store_true")
    ap.add_argument("--emulate-shard", default=None,
                    help="R/N: replay only address shard R of N on this one GPU (scaling projection; "
                         "shards share nothing but the final allgather)")
    ap.add_argument("--granule-log2", type=int, default=3,
                    help="address-shard granule (2^g words; 3 = 64 B of shadow)")
    ap.add_argument("--double-shadow", action="store_true",
                    help="HR_OPT_DOUBLE_SHADOW: reset the previous kernel's shadow on a side stream")
    ap.add_argument("--format", default="c32", choices=["c32", "u64", "pooled"],
                    help="device-resident trace encoding (include/hr.h HR_TRACE_U64 = 256 B/row, C32 = 160 B/row, "
                         "POOLED = the C32 trace re-laid out as warp pools by hr_pool_trace, untimed: for sparse "
                         "address shards)")
    ap.add_argument("--e2e-format", default="packed", choices=["packed", "c32", "u64"],
                    help="host-buffer trace encoding for e2e: packed (HR_TRACE_PACKED, decoded on the device), "
                         "c32 (160 B/row) or u64 (256 B/row)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo lets N ranks share one GPU to test the N>1 path (timings then meaningless)")
    ap.add_argument("--c4-lv", type=int, default=20, help="log2 vertices of the C4 graph for the slowdown")
    ap.add_argument("--clock-ms", type=int, default=100, help="nvidia-smi sampling period during the timed region")
    ap.add_argument("--no-spin", action="store_true", help="default CUDA host-wait scheduling instead of spin")
    ap.add_argument("--sync-report", action="store_true",
                    help="hr_report (host sort/merge, one host round trip per step) instead of hr_report_async")
    ap.add_argument("--no-lazy-reset", action="store_true",
                    help="zero the global shadow at every kernel boundary instead of HR_OPT_LAZY_RESET "
                         "(epoch-tagged words, a real reset every 15 kernels)")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line).
    The sampler is started before the warm-up (its NVML start-up can stall CUDA
    calls for tens of ms) and only samples stamped inside [mark_start, mark_stop]
    are kept."""
    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int, period_ms: int = 100):
        self.idx = gpu_index
        self.period_ms = period_ms
        self.f = tempfile.NamedTemporaryFile(mode="w+", suffix=".csv", delete=False)
        self.p = None
        self.t0 = self.t1 = None

    def start(self):
        if self.period_ms <= 0:
            return
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", str(self.period_ms), "-i", str(self.idx)], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def mark_start(self):
        self.t0 = time.time()

    def mark_stop(self):
        self.t1 = time.time()

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        self.f.seek(0)
        out = self.parse(self.f.read(), self.t0, self.t1)
        os.unlink(self.f.name)
        return out

    @staticmethod
    def parse(text: str, t0=None, t1=None) -> dict:
        """Median SM clock, max clock and throttle reasons of the nvidia-smi
        samples stamped inside [t0, t1] (host epoch seconds; None = all)."""
        import datetime
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in text.splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 10:
                continue
            try:
                ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except ValueError:
                ts = None
            if ts is not None and t0 is not None and not (t0 - 0.05 <= ts <= (t1 or ts) + 0.05):
                continue
            try:
                sm.append(float(parts[2]))
                smax.append(float(parts[3]))
            except ValueError:
                continue
            for n, v in zip(names, parts[6:10]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cuda_spin_wait(local_rank: int) -> bool:
    """Spin-wait scheduling for this process's primary CUDA context (driver API,
    before torch creates the context): a step's host part (hr_report's short
    syncs) then never waits for the OS to wake the thread, which on a busy
    host cost 20-400 ms in a few steps per run."""
    import ctypes
    try:
        cu = ctypes.CDLL("libcuda.so.1")
        if cu.cuInit(0) != 0:
            return False
        dev = ctypes.c_int()
        if cu.cuDeviceGet(ctypes.byref(dev), local_rank) != 0:
            return False
        return cu.cuDevicePrimaryCtxSetFlags(dev, 1) == 0          # CU_CTX_SCHED_SPIN
    except OSError:
        return False


def dist_setup(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dev = local % torch.cuda.device_count()
        torch.cuda.set_device(dev)
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo")
    else:
        torch.cuda.set_device(0)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def _coll_device():
    import torch.distributed as dist
    return "cuda" if dist.get_backend() == "nccl" else "cpu"


def h2d_copy_gbs(nbytes: int = 2 << 30, reps: int = 3) -> float:
    """Plain pinned host->device copy bandwidth of this box (context for e2e,
    which is H2D bound: PCIe rates differ between boxes)."""
    import torch
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        d.copy_(h, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    gbs = nbytes * reps / (e0.elapsed_time(e1) / 1e3) / 1e9
    del h, d
    torch.cuda.empty_cache()
    return gbs


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=_coll_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: int, world: int) -> int:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.int64, device=_coll_device())
    dist.all_reduce(t)
    return int(t.item())


def host_cpu() -> dict:
    """The oracle host: logical CPUs and model (SURVEY §8(d) "Oracle timing")."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:
        usable = os.cpu_count()
    return {"host_cpu_count": os.cpu_count(), "host_cpus_usable": usable, "host_cpu_model": model}


def cpu_baseline(lb: int, seed: int, full_lb: int = 16):
    """The oracle as it stands, single-threaded, on a bounded C5 sample (1/2^(16-lb)
    of the blocks; every block has the same access mix, so the per-access rate
    and the x2^(16-lb) extrapolated full-step time are labelled as such)."""
    import oracle
    from tracegen import c5
    tr = c5.cpu_trace(lb, seed)
    t0 = time.perf_counter()
    res = oracle.check(tr, mode=oracle.BUCKETED)
    dt = time.perf_counter() - t0
    ok = [(r.word, r.scope) for r in res.races] == c5.planted(lb, seed)
    scale = 2 ** (full_lb - lb)
    out = {"value": res.n_accesses / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
           "sample": f"C5 shape at 2^{lb} blocks ({res.n_accesses} accesses, 1/{scale} of the "
                     f"blocks), bucketed mode, {dt:.2f} s; racy set == planted: {ok}",
           "sample_s": dt, "extrapolated_full_step_s": dt * scale,
           "extrapolation": f"x{scale} (EXTRAPOLATED from the 1/{scale} sample, not measured)"}
    out.update(host_cpu())
    return out


def measure_slowdown(dt, kern_ms_launch: float, data_words: int, c4_lv: int):
    """Instrumented vs uninstrumented (SURVEY §8(d) "Slowdown"; paper context:
    7.5x average / 1.08x median over Indigo).  Replay: the check
    kernel vs hrb_raw_replay doing only the raw data accesses of the same
    records.  Online: the same CUDA kernel template with and without hr_check_*."""
    import torch
    from paper_2401_04701_b200 import hirace as hr, online as on
    from tracegen import c4
    out = {}
    data = torch.zeros(data_words, dtype=torch.int32, device="cuda")
    raw_ms = on.time_ms(lambda: on.raw_replay(dt, data, data_words), reps=3, warmup=1)
    out["c5_replay"] = {"checked_kernel_ms": kern_ms_launch, "raw_replay_ms": raw_ms,
                        "slowdown": kern_ms_launch / raw_ms}
    del data
    torch.cuda.empty_cache()
    # C1 (1 block), C3 (1024 blocks), C4 (BFS levels + histogram) online
    d1 = torch.arange(8 * 256 + 8, dtype=torch.int32, device="cuda")
    ck1 = hr.Checker(8 * 256 + 8, 256)
    # instrumented runs reset the report ring each time (a racy kernel would otherwise fill it
    # and every further run would pay the overflow recovery)
    out["c1_online"] = on.slowdown(lambda: on.c1(None, d1, False),
                                   lambda: (hr.hr_reset_report(ck1.ctx), on.c1(ck1.ctx, d1, True)), reps=20)
    ck1.close()
    d3 = torch.randint(0, 100, (2 * 512 * 512,), dtype=torch.int32, device="cuda")
    ck3 = hr.Checker(2 * 512 * 512, 648)
    out["c3_online"] = on.slowdown(lambda: on.c3(None, d3, False),
                                   lambda: (hr.hr_reset_report(ck3.ctx), on.c3(ck3.ctx, d3, True)), reps=10)
    ck3.close()
    g = c4.Graph(c4_lv)
    dev = on.C4Device(g)
    d4 = torch.zeros(g.n + 1024, dtype=torch.int32, device="cuda")
    ck4 = hr.Checker(g.n + 1024, 0, ring_capacity=1 << 24)
    for racy in (False, True):
        out[f"c4_online_{'racy' if racy else 'atomic'}_2^{c4_lv}"] = on.slowdown(
            lambda: dev.run(None, d4, False, racy),
            lambda: (hr.hr_reset_report(ck4.ctx), dev.run(ck4.ctx, d4, True, racy)), reps=5)
    ck4.close()
    for v in out.values():
        for k in list(v):
            v[k] = round(v[k], 4)
    return out


def run_reference(args):
    """--impl reference: the CPU oracle on C5 samples (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    from tracegen import c5
    seed = args.seed if args.seed is not None else c5.DEFAULT_SEED
    tr = c5.cpu_trace(args.ref_lb, seed)
    for _ in range(args.warmup):
        oracle.check(tr)
    t0 = time.perf_counter()
    n = 0
    for _ in range(args.steps):
        n += oracle.check(tr).n_accesses
    dt = time.perf_counter() - t0
    v = n / dt
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic",
        "config": {"workload": f"C5 sample: 2^{args.ref_lb} blocks x 256 threads x 256 accesses "
                               f"(same generator as the GPU arm's 2^{args.lb}-block workload)"},
        "cpu_baseline": dict({"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                              "sample": f"C5 at 2^{args.ref_lb} blocks per step, bucketed single-threaded oracle",
                              "extrapolated_full_step_s": dt / args.steps * 2 ** (args.lb - args.ref_lb),
                              "extrapolation": f"x{2 ** (args.lb - args.ref_lb)} (EXTRAPOLATED, not measured)"},
                             **host_cpu()),
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def run_c3(args):
    """--config c3: C3 (1024 blocks x 256 threads, 2^26 accesses, SMEM shadow)
    on one GPU.  One step = ring reset + replay of the device-resident C32
    trace + hr_report_async.  The SMEM shadow never reaches DRAM, so the
    roofline is instruction issue (bound "alu"): warp instructions per launch
    (ncu smsp__inst_executed.sum of this build, profiles/c3_instructions.json)
    / live kernel time, against 148 SMs x 4 schedulers x 1 warp-instr/clk x
    the max SM clock (B300_MICROARCH.md issue model, B200 SM count)."""
    import numpy as np
    import torch
    from paper_2401_04701_b200 import hirace as hr, online as on
    from tracegen import stencil
    spin = cuda_spin_wait(0) if not args.no_spin else False
    torch.cuda.set_device(0)
    stream = torch.cuda.current_stream().cuda_stream
    removed, n = None, stencil.N                           # the race-free stencil; racy variant below
    tr = stencil.stencil_trace(removed=removed, n=n)
    dt = hr.DeviceTrace.from_trace(tr, compact=True)
    n_acc = int((((tr.rec >> np.uint64(62)) & np.uint64(3)) != 3).sum())
    words, smem = 2 * n * n, 2 * stencil.TILE
    ck = hr.Checker(words, smem, options=hr.HR_OPT_TIMING | args.options)
    blocks = (n // stencil.T) ** 2
    want = []

    def step(replay):
        ck.reset()
        replay()
        ck.report_async()

    clocks = Clocks(0, args.clock_ms)
    clocks.start()
    dev = lambda: ck.replay(dt, stream)  # noqa: E731
    for _ in range(max(args.warmup, 3)):
        step(dev)
    raw, flags = ck.collect_raw()
    parity = [(int(r["kernel"]), int(r["space"]), int(r["block"]), int(r["word"]), int(r["scope"]))
              for r in raw] == want and flags == 0
    hr.hr_replay_timing(ck.ctx)
    hr.hr_launch_count(ck.ctx)
    steps = args.steps
    torch.cuda.synchronize()
    clocks.mark_start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step(dev)
    e1.record()
    torch.cuda.synchronize()
    clocks.mark_stop()
    clk = clocks.stop()
    ms_step = e0.elapsed_time(e1) / steps
    _, _, kern_ms, n_kern = hr.hr_replay_timing(ck.ctx)
    n_launch = hr.hr_launch_count(ck.ctx)
    raw, flags = ck.collect_raw()
    parity = parity and [(int(r["kernel"]), int(r["space"]), int(r["block"]), int(r["word"]), int(r["scope"]))
                         for r in raw] == want
    k_ms = kern_ms / max(n_kern, 1)
    # racy variant (barrier after sweep 20 removed: 524,288 racy shared words per step, so the
    # report — device sort of the ring + 12.6 MB written to pinned host memory — weighs in)
    tr_r = stencil.stencil_trace(removed=20, n=n)
    dt_r = hr.DeviceTrace.from_trace(tr_r, compact=True)
    want_r = [(0, 1, b, int(w), 1) for b in range(blocks) for w in stencil.expected_racy_shared_words(20)]
    rr = lambda: ck.replay(dt_r, stream)  # noqa: E731
    for _ in range(3):
        step(rr)
    ck.collect_raw()
    hr.hr_replay_timing(ck.ctx)
    torch.cuda.synchronize()
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record()
    for _ in range(steps):
        step(rr)
    g1.record()
    torch.cuda.synchronize()
    raw_r, _ = ck.collect_raw()
    _, _, kr_ms, nkr = hr.hr_replay_timing(ck.ctx)
    racy = {"workload": "same stencil, barrier after sweep 20 removed", "ms_per_step": g0.elapsed_time(g1) / steps,
            "value": n_acc / (g0.elapsed_time(g1) / steps / 1e3), "kernel_ms": kr_ms / max(nkr, 1),
            "races_per_step": len(raw_r),
            "parity_vs_closed_form": [(int(r["kernel"]), int(r["space"]), int(r["block"]), int(r["word"]),
                                       int(r["scope"])) for r in raw_r] == want_r}
    del dt_r
    hbm, hbm_kind = peaks()
    sm_max = clk.get("sm_max_mhz") or 1965.0
    issue_peak = 148 * 4 * sm_max * 1e6 / 1e9                          # G warp-instructions/s
    instr, achieved = None, None
    prof = os.path.join(ROOT, "profiles", "c3_instructions.json")
    if os.path.exists(prof):
        pj = json.load(open(prof))
        instr = float(pj["inst_executed_per_launch"])
        achieved = instr / (k_ms / 1e3) / 1e9
    # e2e: the same steps from pinned host buffers (C32 records copied H2D in every step)
    import torch as _t
    pinned = {}
    for name in ("rec32", "recop"):
        x = getattr(dt, name)
        h = _t.empty(x.numel(), dtype=x.dtype, pin_memory=True)
        h.copy_(x)
        pinned[name] = h
    host = type("T", (), {})()
    host.kdesc, host.warp_off, host.rec = dt.kdesc, dt.warp_off.cpu().numpy().view(np.uint64), None
    host.rec32, host.recop = pinned["rec32"].numpy().view(np.uint32), pinned["recop"].numpy()
    h2d = int(host.rec32.nbytes + host.recop.nbytes + host.warp_off.nbytes)
    hrep = lambda: ck.replay_host(host, stream)  # noqa: E731
    for _ in range(2):
        step(hrep)
    ck.collect_raw()
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    for _ in range(steps):
        step(hrep)
    f1.record()
    torch.cuda.synchronize()
    raw_e, _ = ck.collect_raw()
    e2e_ms = f0.elapsed_time(f1) / steps
    parity = parity and len(raw_e) == len(want)
    slow = None
    if not args.no_slowdown:
        d3 = torch.randint(0, 100, (words,), dtype=torch.int32, device="cuda")
        ck3 = hr.Checker(words, smem)
        slow = {"c3_online": on.slowdown(lambda: on.c3(None, d3, False, removed=None),
                                         lambda: on.c3(ck3.ctx, d3, True, removed=None), reps=10)}
        ck3.close()
        data = torch.zeros(words, dtype=torch.int32, device="cuda")
        raw_ms = on.time_ms(lambda: on.raw_replay(dt, data, words), reps=5, warmup=2)
        slow["c3_replay"] = {"checked_kernel_ms": k_ms, "raw_replay_ms": raw_ms, "slowdown": k_ms / raw_ms}
    cpu = None
    if not args.no_cpu:
        import oracle
        small = stencil.stencil_trace(removed=20, n=64)
        t0 = time.perf_counter()
        res = oracle.check(small, mode=oracle.BUCKETED)
        dtc = time.perf_counter() - t0
        cpu = dict({"value": res.n_accesses / dtc, "unit": UNIT, "cores": 1, "kind": "oracle",
                    "sample": f"C3 racy variant at n=64 (16 of the 1024 blocks, {res.n_accesses} accesses), bucketed, "
                              f"{dtc:.2f} s", "extrapolated_full_step_s": dtc * n_acc / res.n_accesses,
                    "extrapolation": "x64 by access count (EXTRAPOLATED, not measured)"}, **host_cpu())
    out = {
        "metric": METRIC, "value": n_acc / (ms_step / 1e3), "unit": UNIT, "n_gpus": 1, "steps": steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": f"C3: shared-memory 2D stencil {n}x{n}, {blocks} blocks x 256 threads, 42 sweeps, "
                               f"race-free (racy variant in racy_variant), {n_acc} checked accesses",
                   "trace_format": "c32", "host_wait": "spin" if spin else "default",
                   "report": "hr_report_async every step", "l2": "trace (0.34 GB) > L2 is streamed; the SMEM "
                   "shadow is per block; no flush needed"},
        "roofline": {"bound": "alu", "achieved": achieved, "peak": issue_peak, "unit": "G warp-instr/s",
                     "frac": (achieved / issue_peak) if achieved else None, "traffic": None,
                     "kernel": "hr_replay_kernel", "kernel_ms": k_ms,
                     "inst_executed_per_launch": instr,
                     "inst_per_warp_row": (instr / (dt.n_rows)) if instr else None,
                     "peak_rule": "148 SMs x 4 SMSPs x 1 warp-instruction/clk x sm_max_mhz",
                     "literal_frac": 8 * n_acc / (k_ms / 1e3) / 1e9 / hbm, "literal_peak_kind": hbm_kind},
        "clocks": clk,
        "e2e": {"value": n_acc / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": 16 + 24 * len(raw_e), "ms_per_step": e2e_ms, "format": "c32"},
        "gpu_launches": n_launch,
        "gpu_launches_detail": {"replay_kernel": n_kern, "all_libhirace": n_launch},
        "racy_variant": racy,
        "slowdown": slow, "cpu_baseline": cpu, "parity_vs_closed_form": parity,
    }
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.config == "c3":
        run_c3(args)
        return
    import numpy as np
    import torch
    from paper_2401_04701_b200 import hirace as hr
    from paper_2401_04701_b200.multigpu import DeviceExchange, exchange_races, shard_owner
    from tracegen import c5

    spin = cuda_spin_wait(int(os.environ.get("LOCAL_RANK", "0"))) if not args.no_spin else False
    rank, world, local = dist_setup(args)
    assert world == args.gpus or world == 1, "launch with torchrun for --gpus > 1"
    emulated = None
    if args.emulate_shard:
        assert world == 1, "--emulate-shard runs one process"
        er, en = (int(x) for x in args.emulate_shard.split("/"))
        emulated = (er, en)
    seed = args.seed if args.seed is not None else c5.DEFAULT_SEED
    lb = args.lb
    stream = torch.cuda.current_stream().cuda_stream

    shard_rank, shard_n = emulated if emulated else (rank, world)
    # --- input: this rank's shard of the trace, generated in HBM (untimed) ---
    if args.format in ("c32", "pooled"):
        rec32, recop, woff, kd = c5.gpu_trace_c32(lb, seed, rank=shard_rank, nshard=shard_n,
                                                  granule_log2=args.granule_log2)
        dt = hr.DeviceTrace(None, woff, kd, rec32, recop)
        n_acc_rank = int(((recop & 3) != 3).sum().item())
    else:
        rec, woff, kd = c5.gpu_trace(lb, seed, rank=shard_rank, nshard=shard_n, granule_log2=args.granule_log2)
        dt = hr.DeviceTrace(rec, woff, kd)
        n_acc_rank = int((((rec >> 62) & 3) != 3).sum().item())
    torch.cuda.synchronize()
    n_rows = dt.n_rows
    # access classes of C5 (tracegen/c5gen.h), for the random-access ceiling (untimed)
    owned, hot_base = c5.total_words(lb) // 2, c5.total_words(lb) - (1 << (lb + 4))
    n_gather = n_own = 0
    n_rec = n_rows * 32
    for c0 in range(0, n_rec, 1 << 27):                   # chunked: no 34 GB temporaries
        c1 = min(n_rec, c0 + (1 << 27))
        if dt.format == hr.HR_TRACE_C32:
            acc_mask = (dt.recop[c0:c1] & 3) != 3
            wv = dt.rec32[c0:c1].to(torch.int64) & 0xFFFFFFFF
        else:
            acc_mask = ((dt.rec[c0:c1] >> 62) & 3) != 3
            wv = dt.rec[c0:c1] & ((1 << 61) - 1)
        n_gather += int((acc_mask & (wv >= owned) & (wv < hot_base)).sum().item())
        n_own += int((acc_mask & (wv < owned)).sum().item())
    del acc_mask, wv
    opts = hr.HR_OPT_TIMING | args.options | (hr.HR_OPT_DOUBLE_SHADOW if args.double_shadow else 0)
    if not (args.no_lazy_reset or args.double_shadow):
        opts |= hr.HR_OPT_LAZY_RESET
    ck = hr.Checker(c5.total_words(lb), 0, shard=(shard_rank, shard_n), options=opts, ring_capacity=1 << 21,
                    granule_log2=args.granule_log2)
    if shard_n > 1:
        dt.flags = hr.HR_TRACE_F_SHARD_OWNED              # the generator kept only this rank's records
    if args.format == "pooled":
        pooled = ck.pool(dt, stream)                      # untimed input re-layout (hr_pool_trace)
        dt.rec32 = dt.recop = None
        rec32 = recop = None  # noqa: F841
        dt = pooled
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        n_rows = dt.n_rows

    step_log = [] if os.environ.get("HR_BENCH_STEPLOG") else None
    # N > 1: device report + allgather of the fixed-size per-rank buffers inside the step, merged
    # on collect; N = 1: device report into pinned host memory
    exchange = DeviceExchange(ck.ctx, 1 << 17) if world > 1 and not args.sync_report else None
    async_report = world == 1 and not args.sync_report

    def step(replay_fn):
        if step_log is not None:                    # diagnostic: where a slow step spends its time
            t0 = time.perf_counter()
            ga, gb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ga.record()
            ck.reset()
            replay_fn()
            gb.record()
            t1 = time.perf_counter()
            gb.synchronize()
            t2 = time.perf_counter()
            raw, flags = ck.report_raw(copy=False)
            t3 = time.perf_counter()
            step_log.append({"issue": round(1e3 * (t1 - t0), 2), "gpu_replay": round(ga.elapsed_time(gb), 2),
                             "wait": round(1e3 * (t2 - t1), 2), "report": round(1e3 * (t3 - t2), 2)})
        elif exchange is not None:
            ck.reset()
            replay_fn()
            exchange.step(stream)                   # a13 on the device + NCCL allgather, no host wait
            return None, None
        elif async_report:
            ck.reset()
            replay_fn()
            ck.report_async()                       # a13 on the device, result -> pinned host memory
            return None, None
        else:
            ck.reset()
            replay_fn()
            raw, flags = ck.report_raw(copy=False)  # view of the reused buffer: no allocation per step
        if world > 1:
            raw, flags = exchange_races(raw, flags)
        return raw, flags

    def collect():
        """The last step's global set (after the loop: off the step's critical path)."""
        if exchange is not None:
            return exchange.collect(fallback_raw=lambda: ck.report_raw())
        return ck.collect_raw()

    dev_replay = lambda: ck.replay(dt, stream)  # noqa: E731

    # clock sampler first: its start-up must not land in the timed region
    clocks = Clocks(torch.cuda.current_device(), args.clock_ms)
    clocks.start()
    # warm-up + correctness of this run against the closed form (planted set)
    for _ in range(max(args.warmup, 1)):
        raw, flags = step(dev_replay)
    if (async_report or exchange is not None) and step_log is None:
        raw, flags = collect()

    def expected():
        pl = c5.planted(lb, seed)
        if emulated:
            return [(w, sc) for w, sc in pl if shard_owner(w >> args.granule_log2, shard_n) == shard_rank]
        return pl

    got = [(int(r["word"]), int(r["scope"])) for r in raw]
    parity_ok = got == expected() and flags == 0
    hr.hr_replay_timing(ck.ctx)                     # drop warm-up launches
    hr.hr_launch_count(ck.ctx)
    # setup objects (torch, traces) out of the collector's way: a full gen-2
    # pass over them inside a host-side report step costs ~10 ms at random
    gc.collect()
    gc.freeze()
    step(dev_replay)                                # one more warm step after the pause
    hr.hr_replay_timing(ck.ctx)
    hr.hr_launch_count(ck.ctx)

    barrier(world)
    torch.cuda.synchronize()
    clocks.mark_start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        raw, flags = step(dev_replay)
    e1.record()
    torch.cuda.synchronize()
    clocks.mark_stop()
    barrier(world)
    clk = clocks.stop()
    ms_total = e0.elapsed_time(e1)
    if step_log is not None:
        print("steplog:", json.dumps(step_log[-args.steps:]), file=sys.stderr)
    reset_ms, n_resets, kern_ms, n_kern = hr.hr_replay_timing(ck.ctx)
    n_launch = hr.hr_launch_count(ck.ctx)
    if (async_report or exchange is not None) and step_log is None:
        raw, flags = collect()                      # the last step's result (pinned host memory / gathered)
    parity_ok = parity_ok and [(int(r["word"]), int(r["scope"])) for r in raw] == expected()

    ms_step = max_over_ranks(ms_total / args.steps, world)
    total_acc = sum_over_ranks(n_acc_rank, world)
    value = total_acc / (ms_step / 1e3)
    kern_ms_launch = max_over_ranks(kern_ms / max(n_kern, 1), world)
    reset_ms_step = max_over_ranks(reset_ms / args.steps, world)     # lazy reset: not every step resets

    # roofline of the dominant kernel (the replay), rank 0's launch
    peak, peak_kind = peaks()
    algo_bytes = dt.record_bytes() + BYTES_PER_ACCESS_ALGO * n_acc_rank
    achieved = algo_bytes / (kern_ms / max(n_kern, 1) / 1e3) / 1e9
    traffic = None
    l2_atomic = None
    prof = os.path.join(ROOT, "profiles", "replay_dram_bytes.json")
    rates_path = os.path.join(ROOT, "profiles", "b200_access_rates.json")
    if os.path.exists(prof):
        try:
            pj = json.load(open(prof))
            if world == 1 and int(pj.get("lb", -1)) == lb and pj.get("format", "u64") == args.format \
                    and not emulated:
                traffic = float(pj["dram_bytes_per_launch"])
                if "l2_atom_cas_requests_per_launch" in pj and os.path.exists(rates_path):
                    # north_star: "L2 atomic throughput against the chip's peak" — committed + failed
                    # CAS requests the L2 served per second of the live launch, against the measured
                    # L2 atomic unit rate (random 64-bit CAS on an L2-resident set)
                    ops = float(pj["l2_atom_cas_requests_per_launch"])
                    rl2 = json.load(open(rates_path))["random_cas_l2_per_s"]
                    ach = ops / (kern_ms / max(n_kern, 1) / 1e3)
                    l2_atomic = {"ops_per_launch": ops, "achieved_per_s": ach, "peak_per_s": rl2,
                                 "frac": ach / rl2, "unit": "CAS/s",
                                 "source": "ncu lts__t_requests_srcunit_tex_op_atom_dot_cas.sum of the same "
                                           "launch (profiles/replay_dram_bytes.json); peak = measured random "
                                           "64-bit CAS rate on an L2-resident set (profiles/b200_access_rates.json)"}
        except Exception:
            traffic = None
    literal = BYTES_PER_ACCESS_LITERAL * total_acc / (ms_step / 1e3) / 1e9 / (peak * world)
    # the floor that actually binds C5: random 8-byte RMWs on cold HBM words run at
    # the measured DRAM random-access rate, the rest streams at the copy peak
    ceiling = None
    if os.path.exists(rates_path):
        rates = json.load(open(rates_path))
        floor_ms = 1e3 * (n_gather / rates["random_cas_hbm_per_s"] +
                          (dt.record_bytes() + BYTES_PER_ACCESS_ALGO * n_own) / (peak * 1e9))
        ceiling = {"kind": "measured random-DRAM RMW rate + copy peak", "rate_source": os.path.relpath(rates_path, ROOT),
                   "random_gathers": n_gather, "coalesced_own_row": n_own,
                   "floor_ms_per_launch": floor_ms, "kernel_ms": kern_ms / max(n_kern, 1),
                   "frac_of_floor": floor_ms / (kern_ms / max(n_kern, 1))}

    slow = None
    if rank == 0 and world == 1 and not args.no_slowdown:
        slow = measure_slowdown(dt, kern_ms / max(n_kern, 1), c5.total_words(lb), args.c4_lv)

    # --- e2e through the C ABI with HOST buffers ---
    e2e = None
    if not args.no_e2e and args.e2e_format == "packed":
        # pack the u64 trace on the device (untimed), keep only the pinned host copy
        src = dt
        if dt.format != hr.HR_TRACE_U64:
            dt.rec = dt.rec32 = dt.recop = None
            rec32 = recop = None  # noqa: F841
            grec, _, _ = c5.gpu_trace(lb, seed, rank=shard_rank, nshard=shard_n, granule_log2=args.granule_log2)
            src = hr.DeviceTrace(grec, woff, kd)
            grec = None  # noqa: F841
        pk = ck.pack(src, stream)
        host_trace = pk.to_host()
        src = pk = None
        dt.rec = dt.rec32 = dt.recop = None
        rec = None  # noqa: F841
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        h2d = int(host_trace.packed.nbytes + host_trace.pack_off.nbytes + host_trace.warp_off.nbytes)
    elif not args.no_e2e:
        host_trace = type("T", (), {})()
        host_trace.kdesc = kd
        host_trace.warp_off = woff.cpu().numpy().view(np.uint64)
        dt.rec = dt.rec32 = dt.recop = None                 # free the device trace: staging replaces it
        rec = rec32 = recop = None  # noqa: F841
        torch.cuda.empty_cache()
        pinned = []
        if args.e2e_format == "c32":
            g32, gop, _, _ = c5.gpu_trace_c32(lb, seed, rank=shard_rank, nshard=shard_n,
                                              granule_log2=args.granule_log2)
            parts = (("rec32", g32), ("recop", gop))
            host_trace.rec = None
        else:
            grec, _, _ = c5.gpu_trace(lb, seed, rank=shard_rank, nshard=shard_n, granule_log2=args.granule_log2)
            parts = (("rec", grec),)
            host_trace.rec32 = None
        for name, tsr in parts:
            h = torch.empty(tsr.numel(), dtype=tsr.dtype, pin_memory=True)
            h.copy_(tsr)
            pinned.append(h)
            arr = h.numpy()
            setattr(host_trace, name, arr.view(np.uint64) if name == "rec" else arr)
        parts = g32 = gop = grec = None  # noqa: F841
        torch.cuda.empty_cache()
        h2d = sum(int(h.numel() * h.element_size()) for h in pinned) + int(host_trace.warp_off.nbytes)
    if not args.no_e2e:
        h2d_probe = h2d_copy_gbs()                      # this box's plain pinned H2D rate (untimed)
        host_replay = lambda: ck.replay_host(host_trace, stream)  # noqa: E731
        for _ in range(args.warmup):
            step(host_replay)
        barrier(world)
        torch.cuda.synchronize()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(args.steps):
            raw_e, _ = step(host_replay)
        f1.record()
        torch.cuda.synchronize()
        if (async_report or exchange is not None) and step_log is None:
            raw_e, _ = collect()
        barrier(world)
        e2e_ms = max_over_ranks(f0.elapsed_time(f1) / args.steps, world)
        parity_ok = parity_ok and [(int(r["word"]), int(r["scope"])) for r in raw_e] == expected()
        e2e = {"value": total_acc / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "h2d_achieved_gbs": h2d / (e2e_ms / 1e3) / 1e9, "h2d_copy_probe_gbs": h2d_probe,
               "d2h_bytes_per_step": int(16 + 24 * len(raw_e) // max(world, 1)),
               "ms_per_step": e2e_ms, "format": args.e2e_format}
        hr.hr_replay_timing(ck.ctx)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args.cpu_lb, seed)

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": f"C5: {total_acc} checked accesses (2^{lb} blocks x 256 threads x 256), "
                                   f"global trace over 2^{lb + 16} words, address-sharded (rotated granule stripes, x{world})",
                       "trace_format": args.format, "host_wait": "spin" if spin else "default",
                       "report": ("hr_report_async: device sort/merge, result written to pinned host memory "
                                  "every step, collected after the loop" if async_report else
                                  "hr_report_async_to into a device buffer + NCCL all_gather_into_tensor of the "
                                  "2^17-record per-rank buffers every step (no host round trip); merged with "
                                  "hr_merge_races after the loop" if exchange is not None else
                                  "hr_report: host round trip per step"),
                       "kernel_boundary_reset": ("memset per kernel" if (args.no_lazy_reset or args.double_shadow)
                                                 else "lazy: epoch-tagged shadow words, a real memset every 15 "
                                                      "kernels (4.65 ms at C5, ~0.31 ms per step amortized; a 5-step "
                                                      "window holds 0 or 1 of them, see shadow_resets_in_timed_steps)"),
                       "parallelism": f"address-shard x{world}", "l2": "inputs larger than L2 "
                       "(trace + shadow >> 126 MB; no flush needed)", "seed": seed},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                         "kernel": "hr_replay_kernel", "kernel_ms": kern_ms / max(n_kern, 1),
                         "algo_bytes_per_launch": algo_bytes,
                         "algo_bytes_rule": f"records ({args.format}: {dt.record_bytes() // max(n_rows, 1)} B/row) "
                                            "+ 16 B shadow RMW per checked access",
                         "l2_atomic": l2_atomic},
            "paper_context": {
                "note": "the paper's own numbers on its RTX 2070 Super (PAPER.md:796-803): context, not targets",
                "speedup_vs_iguard": ">10x faster on average than iGUARD over 580 kernels (PAPER.md:86)",
                "memory_overhead": "8 B of shadow per monitored word vs iGUARD's 16 B: half (PAPER.md:725, 927)",
                "slowdown": "7.5x average, 1.08x median over 5,105 executions (PAPER.md:898)"},
            "literal_roofline_frac": literal,
            "ceiling": ceiling,
            "step_breakdown_ms": {"replay_kernel": kern_ms_launch,
                                  "shadow_reset" + (" (side stream, overlapped)" if args.double_shadow else ""):
                                      reset_ms_step,
                                  "shadow_resets_in_timed_steps": n_resets,
                                  "rest(report,ring reset,exchange)":
                                      ms_step - kern_ms_launch - (0.0 if args.double_shadow else reset_ms_step)},
            "clocks": clk,
            "e2e": e2e,
            "gpu_launches": n_launch,
            "gpu_launches_detail": {"replay_kernel": n_kern, "all_libhirace": n_launch,
                                    "rule": "every libhirace kernel launched in the timed region: the replay, "
                                            "the end-of-kernel spill scan (a9 overflow recovery; returns at once "
                                            "unless the ring overflowed), "
                                            + ("the report's key / head / emit kernels, its 2 CUB radix sorts "
                                               "(2 + one pass per 8 key bits that can be set) and CUB scan (2)"
                                               if (async_report or exchange is not None) else
                                               "the report's key / gather kernels and its 2 CUB radix sorts "
                                               "(10 kernels each)")},
            "slowdown": slow,
            "cpu_baseline": cpu,
            "parity_vs_closed_form": parity_ok,
        }
        if emulated:
            out["emulated_shard"] = {"rank": shard_rank, "of": shard_n, "shard_accesses": total_acc,
                                     "shard_ms_per_step": ms_step,
                                     "note": "one shard replayed alone on one GPU: a projection of the N-GPU "
                                             "step (ranks share nothing but the final allgather), not a "
                                             "multi-GPU measurement"}
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
