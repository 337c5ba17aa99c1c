"""Binding of include/hr_bench.h: the online-instrumented C1 / C3 / C4 kernels
(plain and instrumented builds of the same CUDA templates) and the paper's
instrumented-vs-uninstrumented slowdown.  Marshalling
only; the kernels live in libhirace.so."""
from __future__ import annotations

import ctypes
from typing import Dict, Optional

import numpy as np

from . import hirace

EXPORTS = ("hrb_c1", "hrb_c1_array", "hrb_c3", "hrb_c4_level", "hrb_c4_hist", "hrb_raw_replay", "hrb_masked_sync")


def _lib():
    lib = hirace.load()
    if not getattr(lib, "_hrb_ready", False):
        vp, i, u32 = ctypes.c_void_p, ctypes.c_int, ctypes.c_uint32
        lib.hrb_c1.argtypes = [vp, i, u32, i, i, vp, vp]
        lib.hrb_c1_array.argtypes = [vp, u32, i, i, vp, vp]
        lib.hrb_c3.argtypes = [vp, i, u32, i, i, i, vp, vp]
        lib.hrb_c4_level.argtypes = [vp, i, u32, i, u32, vp, vp, vp, i, vp, vp]
        lib.hrb_c4_hist.argtypes = [vp, i, u32, i, u32, vp, vp, vp]
        lib.hrb_raw_replay.argtypes = [ctypes.POINTER(hirace.HrTrace), vp, ctypes.c_uint64, vp]
        lib.hrb_masked_sync.argtypes = [vp, u32, vp, vp]
        for n in EXPORTS:
            getattr(lib, n).restype = ctypes.c_int
        lib._hrb_ready = True
    return lib


def _stream():
    import torch
    return torch.cuda.current_stream().cuda_stream


def _ok(rc, ctx, what):
    hirace._check(rc, ctx, what)


C1_REMOVED = {None: -1, "load": 0}


def c1(ctx, data, instrumented: bool, removed=32, rounds: int = 8, kernel_id: int = 0):
    r = C1_REMOVED.get(removed, removed)
    _ok(_lib().hrb_c1(ctx, int(instrumented), kernel_id, rounds, r, data.data_ptr(), _stream()), ctx, "hrb_c1")


def c1_array(ctx, data, removed=32, rounds: int = 8, kernel_id: int = 0):
    """C1 through the hr_array<T> wrapper (transparent instrumentation)."""
    r = C1_REMOVED.get(removed, removed)
    _ok(_lib().hrb_c1_array(ctx, kernel_id, rounds, r, data.data_ptr(), _stream()), ctx, "hrb_c1_array")


def c3(ctx, data, instrumented: bool, n: int = 512, sweeps: int = 42, removed: Optional[int] = 20,
       kernel_id: int = 0):
    r = -1 if removed is None else removed
    _ok(_lib().hrb_c3(ctx, int(instrumented), kernel_id, n, sweeps, r, data.data_ptr(), _stream()), ctx, "hrb_c3")


def masked_sync(ctx, data, kernel_id: int = 0):
    """The sub-warp __syncwarp(mask) kernel (include/hr_bench.h hrb_masked_sync)."""
    _ok(_lib().hrb_masked_sync(ctx, kernel_id, data.data_ptr(), _stream()), ctx, "hrb_masked_sync")


def raw_replay(dtrace, data, data_words: int):
    """Uninstrumented replay of a hirace.DeviceTrace (the slowdown denominator)."""
    t = dtrace.c()
    _ok(_lib().hrb_raw_replay(ctypes.byref(t), data.data_ptr(), data_words, _stream()), None, "hrb_raw_replay")


class C4Device:
    """The C4 graph (CSR + final BFS levels) resident on the GPU."""

    def __init__(self, graph, device="cuda"):
        import torch
        rp, col, lvl = graph.csr()
        self.n = graph.n
        self.n_levels = graph.n_levels
        self.rp = torch.from_numpy(rp.view(np.int64)).to(device)
        self.col = torch.from_numpy(col.view(np.int32)).to(device)
        self.flevel = torch.from_numpy(lvl).to(device)

    def run(self, ctx, data, instrumented: bool, racy: bool, kernel_base: int = 0):
        """All BFS levels then the histogram, as separate kernels (kernel ids
        kernel_base + level, histogram last) — the same kernels as tracegen.c4."""
        lib = _lib()
        s = _stream()
        for L in range(self.n_levels):
            _ok(lib.hrb_c4_level(ctx, int(instrumented), kernel_base + L, int(racy), self.n, self.rp.data_ptr(),
                                 self.col.data_ptr(), self.flevel.data_ptr(), L, data.data_ptr(), s),
                ctx, "hrb_c4_level")
        _ok(lib.hrb_c4_hist(ctx, int(instrumented), kernel_base + self.n_levels, int(racy), self.n,
                            self.rp.data_ptr(), data.data_ptr(), s), ctx, "hrb_c4_hist")


def time_ms(fn, reps: int = 5, warmup: int = 2) -> float:
    """Median device time of fn() over reps, CUDA events on the current stream."""
    import torch
    for _ in range(warmup):
        fn()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def slowdown(plain_fn, instr_fn, reps: int = 5) -> Dict[str, float]:
    p = time_ms(plain_fn, reps)
    i = time_ms(instr_fn, reps)
    return {"plain_ms": p, "instrumented_ms": i, "slowdown": i / p}
