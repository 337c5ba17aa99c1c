"""Thin Python binding of the C ABI in include/hr.h (argument marshalling only).

Every step of the check runs in libhirace.so (sm_100a).  PyTorch provides
device memory, streams and (in ``multigpu``) process groups.  There is no CPU
fallback: if the library cannot be loaded this module raises on import.

Function names mirror the C ABI: ``hr_init``, ``hr_set_shard``,
``hr_shadow_alloc``, ``hr_kernel_begin``, ``hr_replay_trace``,
``hr_replay_trace_host``, ``hr_report``, ``hr_reset_report``, ``hr_counters``,
``hr_fsm_table``, ``hr_last_error``, ``hr_destroy``.  ``Checker`` bundles them
for tests and bench.py.
"""
from __future__ import annotations

import ctypes
import os
from typing import List, NamedTuple, Optional, Tuple

import numpy as np

from . import build as _build

HR_OK, HR_E_ARG, HR_E_NOMEM, HR_E_CUDA, HR_E_STATE, HR_E_INCOMPLETE = 0, -1, -2, -3, -4, -5
HR_GLOBAL, HR_SHARED = 0, 1
HR_F_CLOCK_OVERFLOW, HR_F_RING_OVERFLOW, HR_F_MODEL_VIOLATION = 1, 2, 4
HR_F_BARRIER_DIVERGENCE, HR_F_UNMONITORED, HR_F_INCOMPLETE = 8, 16, 32
HR_OPT_NO_COALESCE, HR_OPT_NO_FASTEXIT, HR_OPT_TIMING, HR_OPT_NO_SPECULATE, HR_OPT_NO_POOL, HR_OPT_POOL = \
    1, 2, 4, 8, 16, 32
HR_OPT_DOUBLE_SHADOW = 64
HR_OPT_FINITE_HISTORY = 128
HR_OPT_POOL_WIDE = 256
HR_OPT_ROW_WIDE = 512
HR_OPT_NO_COMPACT = 1024
HR_OPT_SPECULATE = 2048
HR_OPT_SMEM32 = 4096
HR_OPT_LAZY_RESET = 8192
HR_OPT_BSERIAL = 16384
HR_OPT_ROW_NARROW = 65536
HR_OPT_NO_STREAMS = 131072
HR_OPT_BINNED = 262144
HR_OPT_NO_BINNED = 524288
HR_OPT_HYBRID = 1048576
HR_OPT_BIN_ALL = 2097152
EXPORTS = ("hr_init", "hr_set_shard", "hr_set_shard_ex", "hr_set_representatives", "hr_set_warp_tile", "hr_shadow_alloc", "hr_kernel_begin", "hr_replay_trace",
           "hr_replay_trace_host", "hr_pack_trace", "hr_unpack_trace", "hr_pool_trace", "hr_report", "hr_report_async",
           "hr_report_async_to",
           "hr_report_collect", "hr_merge_races", "hr_race_classes", "hr_reset_report", "hr_counters",
           "hr_replay_timing", "hr_launch_count",
           "hr_fsm_table",
           "hr_device_view", "hr_last_error", "hr_destroy")


class HrConfig(ctypes.Structure):
    _fields_ = [("state_bits", ctypes.c_uint8), ("tid_bits", ctypes.c_uint8), ("bc_bits", ctypes.c_uint8),
                ("wc_bits", ctypes.c_uint8), ("ring_capacity", ctypes.c_uint32), ("device", ctypes.c_int),
                ("options", ctypes.c_uint32), ("spill_capacity", ctypes.c_uint32)]


class HrRace(ctypes.Structure):
    _fields_ = [("word", ctypes.c_uint64), ("block", ctypes.c_uint32), ("kernel", ctypes.c_uint32),
                ("first_tid", ctypes.c_uint32), ("space", ctypes.c_uint8), ("scope", ctypes.c_uint8),
                ("first_kind", ctypes.c_uint8), ("prev_state", ctypes.c_uint8)]


HR_TRACE_U64, HR_TRACE_C32, HR_TRACE_PACKED, HR_TRACE_POOLED = 0, 1, 2, 3
HR_TRACE_F_SHARD_OWNED = 1


class HrTrace(ctypes.Structure):
    _fields_ = [("rec", ctypes.c_void_p), ("n_rows", ctypes.c_uint64), ("kdesc", ctypes.c_void_p),
                ("n_kernels", ctypes.c_uint32), ("kernel_base", ctypes.c_uint32),
                ("warp_off", ctypes.c_void_p), ("n_warp_off", ctypes.c_uint64),
                ("format", ctypes.c_uint32), ("flags", ctypes.c_uint32),
                ("rec32", ctypes.c_void_p), ("recop", ctypes.c_void_p),
                ("packed", ctypes.c_void_p), ("pack_off", ctypes.c_void_p)]


assert ctypes.sizeof(HrRace) == 24

_lib = None


def load(build_if_missing: bool = True) -> ctypes.CDLL:
    """Load libhirace.so (built in-tree by __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("HIRACE_LIB", _build.LIB)   # variant builds for A/B measurements
    if not os.path.exists(path):
        if not build_if_missing:
            raise ImportError(f"{path} missing: run __graft_entry__.build()")
        _build.build()
    lib = ctypes.CDLL(path)
    P = ctypes.POINTER
    vp = ctypes.c_void_p
    sig = {
        "hr_init": ([P(HrConfig), P(vp)], ctypes.c_int),
        "hr_set_shard": ([vp, ctypes.c_uint32, ctypes.c_uint32], ctypes.c_int),
        "hr_set_representatives": ([vp, ctypes.c_uint32, ctypes.c_uint32], ctypes.c_int),
        "hr_set_warp_tile": ([vp, ctypes.c_uint32], ctypes.c_int),
        "hr_set_shard_ex": ([vp, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32], ctypes.c_int),
        "hr_shadow_alloc": ([vp, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, P(vp)], ctypes.c_int),
        "hr_kernel_begin": ([vp, vp], ctypes.c_int),
        "hr_replay_trace": ([vp, P(HrTrace), vp], ctypes.c_int),
        "hr_replay_trace_host": ([vp, P(HrTrace), vp], ctypes.c_int),
        "hr_pack_trace": ([vp, P(HrTrace), vp, ctypes.c_uint64, vp, P(ctypes.c_uint64), vp], ctypes.c_int),
        "hr_unpack_trace": ([vp, P(HrTrace), vp, vp], ctypes.c_int),
        "hr_pool_trace": ([vp, P(HrTrace), vp, vp, ctypes.c_uint64, vp, P(ctypes.c_uint64), vp], ctypes.c_int),
        "hr_report": ([vp, P(HrRace), ctypes.c_size_t, P(ctypes.c_size_t), P(ctypes.c_uint32)], ctypes.c_int),
        "hr_merge_races": ([vp, ctypes.c_size_t, vp, ctypes.c_size_t, P(ctypes.c_size_t)], ctypes.c_int),
        "hr_report_async": ([vp, vp], ctypes.c_int),
        "hr_report_async_to": ([vp, vp, vp, ctypes.c_uint32, vp], ctypes.c_int),
        "hr_report_collect": ([vp, P(HrRace), ctypes.c_size_t, P(ctypes.c_size_t), P(ctypes.c_uint32)], ctypes.c_int),
        "hr_race_classes": ([vp, P(HrTrace), vp, ctypes.c_size_t, vp, vp], ctypes.c_int),
        "hr_reset_report": ([vp], ctypes.c_int),
        "hr_counters": ([vp, P(ctypes.c_uint64)], ctypes.c_int),
        "hr_launch_count": ([vp, P(ctypes.c_uint64)], ctypes.c_int),
        "hr_replay_timing": ([vp, P(ctypes.c_double), P(ctypes.c_uint64), P(ctypes.c_double),
                              P(ctypes.c_uint64)], ctypes.c_int),
        "hr_fsm_table": ([P(ctypes.c_uint8), P(ctypes.c_uint8)], ctypes.c_int),
        "hr_device_view": ([vp, vp, ctypes.c_size_t], ctypes.c_int),
        "hr_last_error": ([vp], ctypes.c_char_p),
        "hr_destroy": ([vp], None),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


class HiraceError(RuntimeError):
    def __init__(self, msg: str, status: int = 0):
        super().__init__(msg)
        self.status = status


def _check(rc: int, ctx=None, what: str = ""):
    if rc != HR_OK:
        msg = load().hr_last_error(ctx).decode() if ctx else ""
        raise HiraceError(f"{what} failed with status {rc}: {msg}", rc)


# ---- C-ABI mirrors -------------------------------------------------------------

def hr_init(bc_bits: int = 16, wc_bits: int = 16, ring_capacity: int = 1 << 20, device: int = 0,
            options: int = 0, spill_capacity: int = 0):
    """spill_capacity 0 = automatic (include/hr.h, hr_config)."""
    cfg = HrConfig(5, 27, bc_bits, wc_bits, ring_capacity, device, options, spill_capacity)
    ctx = ctypes.c_void_p()
    _check(load().hr_init(ctypes.byref(cfg), ctypes.byref(ctx)), None, "hr_init")
    return ctx


def hr_set_shard(ctx, rank: int, count: int, granule_log2: int = 3):
    _check(load().hr_set_shard_ex(ctx, rank, count, granule_log2), ctx, "hr_set_shard_ex")


def hr_set_representatives(ctx, block_stride: int = 1, warp_stride: int = 1):
    """Check only blocks % block_stride == 0 and warps % warp_stride == 0."""
    _check(load().hr_set_representatives(ctx, block_stride, warp_stride), ctx, "hr_set_representatives")


def hr_set_warp_tile(ctx, tile_log2: int):
    """Online kernels' warp-level barriers are tiles of 2^tile_log2 lanes (0/5 = whole warps; reading R8)."""
    _check(load().hr_set_warp_tile(ctx, tile_log2), ctx, "hr_set_warp_tile")


def hr_shadow_alloc(ctx, space: int, base_word: int, n_words: int) -> int:
    region = ctypes.c_void_p()
    _check(load().hr_shadow_alloc(ctx, space, base_word, n_words, ctypes.byref(region)), ctx,
           "hr_shadow_alloc")
    return region.value or 0


def hr_kernel_begin(ctx, stream: int = 0):
    _check(load().hr_kernel_begin(ctx, ctypes.c_void_p(stream)), ctx, "hr_kernel_begin")


def hr_replay_trace(ctx, t: HrTrace, stream: int = 0):
    _check(load().hr_replay_trace(ctx, ctypes.byref(t), ctypes.c_void_p(stream)), ctx, "hr_replay_trace")


def hr_replay_trace_host(ctx, t: HrTrace, stream: int = 0):
    _check(load().hr_replay_trace_host(ctx, ctypes.byref(t), ctypes.c_void_p(stream)), ctx,
           "hr_replay_trace_host")


def hr_pack_trace(ctx, t: HrTrace, out: int, cap: int, pack_off: int, stream: int = 0) -> int:
    """Encode a device U64 trace as HR_TRACE_PACKED; out == 0 is the size query.
    Returns the packed size in bytes (with the 16-byte slack)."""
    n = ctypes.c_uint64()
    _check(load().hr_pack_trace(ctx, ctypes.byref(t), ctypes.c_void_p(out or None), cap, ctypes.c_void_p(pack_off),
                                ctypes.byref(n), ctypes.c_void_p(stream)), ctx, "hr_pack_trace")
    return int(n.value)


def hr_pool_trace(ctx, t: HrTrace, rec_out: int, tag_out: int, cap_rows: int, woff_out: int,
                  stream: int = 0) -> int:
    """Re-lay a device U64/C32 trace as HR_TRACE_POOLED; rec_out == 0 is the
    size query.  Returns the pooled row count."""
    n = ctypes.c_uint64()
    _check(load().hr_pool_trace(ctx, ctypes.byref(t), ctypes.c_void_p(rec_out or None), ctypes.c_void_p(tag_out or None),
                                cap_rows, ctypes.c_void_p(woff_out or None), ctypes.byref(n), ctypes.c_void_p(stream)),
           ctx, "hr_pool_trace")
    return int(n.value)


def hr_unpack_trace(ctx, t: HrTrace, rec_out: int, stream: int = 0):
    _check(load().hr_unpack_trace(ctx, ctypes.byref(t), ctypes.c_void_p(rec_out), ctypes.c_void_p(stream)), ctx,
           "hr_unpack_trace")


class Race(NamedTuple):
    kernel: int
    space: int
    block: int
    word: int
    scope: int


RACE_DTYPE = np.dtype([("word", "<u8"), ("block", "<u4"), ("kernel", "<u4"), ("first_tid", "<u4"),
                       ("space", "u1"), ("scope", "u1"), ("first_kind", "u1"), ("prev_state", "u1")])
assert RACE_DTYPE.itemsize == 24


_report_buf: Optional[np.ndarray] = None


def _report_into(fn, ctx, cap: int, copy: bool, what: str) -> Tuple[np.ndarray, int]:
    global _report_buf
    while True:
        if _report_buf is None or _report_buf.shape[0] < cap:
            _report_buf = np.empty(cap, dtype=RACE_DTYPE)
        buf = _report_buf
        cap = buf.shape[0]
        n = ctypes.c_size_t(0)
        fl = ctypes.c_uint32(0)
        rc = fn(ctx, buf.ctypes.data_as(ctypes.POINTER(HrRace)), cap, ctypes.byref(n), ctypes.byref(fl))
        if rc == HR_E_ARG and n.value > cap:
            if what == "hr_report_collect":      # the result stays in the ctx's pinned buffer: re-read it
                fn = load().hr_report
            cap = int(n.value)
            continue
        _check(rc, ctx, what)
        return (buf[: n.value].copy() if copy else buf[: n.value]), int(fl.value)


def hr_report_raw(ctx, cap: int = 1 << 17, copy: bool = True) -> Tuple[np.ndarray, int]:
    """(sorted unique race records as a structured array of hr_race, flags).
    The staging buffer is reused between calls; the result is a copy unless
    copy=False (then a view valid until the next call: no allocation, no
    page faults in a timed loop)."""
    return _report_into(load().hr_report, ctx, cap, copy, "hr_report")


def hr_report_async(ctx, stream: Optional[int] = None):
    """Enqueue the device-side report (hr_report_async); no host wait."""
    _check(load().hr_report_async(ctx, stream or None), ctx, "hr_report_async")


def hr_report_async_to(ctx, out_ptr: int, out_cap: int, hdr_ptr: int, stream: Optional[int] = None):
    """Enqueue the device-side report into caller DEVICE buffers: out (out_cap
    hr_race records) and hdr (4 uint32: unique count, flags, raw count,
    overflow).  No host wait (include/hr.h)."""
    _check(load().hr_report_async_to(ctx, stream or None, ctypes.c_void_p(out_ptr), out_cap,
                                     ctypes.c_void_p(hdr_ptr)), ctx, "hr_report_async_to")


def hr_report_collect(ctx, cap: int = 1 << 17, copy: bool = True) -> Tuple[np.ndarray, int]:
    """Wait for the last hr_report_async; same result as hr_report_raw."""
    return _report_into(load().hr_report_collect, ctx, cap, copy, "hr_report_collect")


def hr_merge_races(parts: np.ndarray) -> np.ndarray:
    """Sorted unique union of race records (hr_race structured array), e.g. the
    concatenated per-shard reports after an allgather.  Host-only C call."""
    src = np.ascontiguousarray(parts, dtype=RACE_DTYPE)
    out = np.empty(max(len(src), 1), dtype=RACE_DTYPE)
    n = ctypes.c_size_t(0)
    _check(load().hr_merge_races(src.ctypes.data if len(src) else None, len(src), out.ctypes.data, len(out),
                                 ctypes.byref(n)), None, "hr_merge_races")
    return out[: n.value]


def races_of(raw: np.ndarray) -> List[Race]:
    return [Race(int(r["kernel"]), int(r["space"]), int(r["block"]), int(r["word"]), int(r["scope"]))
            for r in raw]


def hr_report(ctx, cap: int = 1 << 17) -> Tuple[List[Race], int, np.ndarray]:
    """(sorted unique races as (kernel, space, block, word, scope), flags, raw records)."""
    raw, flags = hr_report_raw(ctx, cap)
    return races_of(raw), flags, raw


def hr_race_classes(ctx, t: HrTrace, raw: np.ndarray, stream: int = 0) -> np.ndarray:
    """Class mask per race record of `raw` (bit0 W-W, bit1 R-W, bit2 A-W, bit3 A-R)."""
    raw = np.ascontiguousarray(raw)
    out = np.zeros(len(raw), dtype=np.uint8)
    _check(load().hr_race_classes(ctx, ctypes.byref(t), raw.ctypes.data, len(raw), out.ctypes.data,
                                  ctypes.c_void_p(stream)), ctx, "hr_race_classes")
    return out


def hr_reset_report(ctx):
    _check(load().hr_reset_report(ctx), ctx, "hr_reset_report")


def hr_counters(ctx) -> List[int]:
    out = (ctypes.c_uint64 * 4)()
    _check(load().hr_counters(ctx, out), ctx, "hr_counters")
    return list(out)


def hr_replay_timing(ctx) -> Tuple[float, int, float, int]:
    """(reset ms, resets, kernel ms, kernels) since the last call (HR_OPT_TIMING)."""
    a, b, c, d = ctypes.c_double(), ctypes.c_uint64(), ctypes.c_double(), ctypes.c_uint64()
    _check(load().hr_replay_timing(ctx, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c), ctypes.byref(d)),
           ctx, "hr_replay_timing")
    return a.value, int(b.value), c.value, int(d.value)


def hr_launch_count(ctx) -> int:
    """Kernels the ctx launched since the last call (CUB scans and sorts counted by their kernels)."""
    n = ctypes.c_uint64()
    _check(load().hr_launch_count(ctx, ctypes.byref(n)), ctx, "hr_launch_count")
    return int(n.value)


def hr_fsm_table() -> Tuple[bytes, bytes]:
    t = (ctypes.c_uint8 * 2048)()
    f = (ctypes.c_uint8 * 32)()
    _check(load().hr_fsm_table(t, f), None, "hr_fsm_table")
    return bytes(t), bytes(f)


def hr_last_error(ctx) -> str:
    return load().hr_last_error(ctx).decode()


def hr_destroy(ctx):
    load().hr_destroy(ctx)


# ---- convenience wrapper -----------------------------------------------------------

class DeviceTrace:
    """A trace resident in HBM: torch tensors for the records and warp offsets,
    host kdesc.  U64 format: ``rec`` int64 (n_rows*32).  C32 format: ``rec32``
    int32 and ``recop`` uint8 (op | space<<2), both n_rows*32.  PACKED format:
    ``packed`` uint8 and ``pack_off`` int64 (made by ``Checker.pack``)."""

    def __init__(self, rec, warp_off, kdesc: np.ndarray, rec32=None, recop=None, packed=None, pack_off=None,
                 n_rows: Optional[int] = None, pooled: bool = False):
        self.rec, self.rec32, self.recop = rec, rec32, recop
        self.packed, self.pack_off = packed, pack_off
        self.warp_off = warp_off
        self.kdesc = np.ascontiguousarray(kdesc, dtype=np.uint64)
        self.flags = 0                          # HR_TRACE_F_* (e.g. SHARD_OWNED for a per-rank shard)
        if pooled:                              # rec: pooled entries, recop: their simulated lanes
            self.format = HR_TRACE_POOLED
            self.n_rows = rec.numel() // 32
        elif packed is not None:
            self.format = HR_TRACE_PACKED
            self.n_rows = int(n_rows)
        else:
            self.format = HR_TRACE_C32 if rec32 is not None else HR_TRACE_U64
            self.n_rows = (rec32.numel() if rec32 is not None else rec.numel()) // 32

    @staticmethod
    def from_trace(trace, device="cuda", compact: bool = False) -> "DeviceTrace":
        import torch
        wo = torch.from_numpy(np.ascontiguousarray(trace.warp_off).view(np.int64)).to(device)
        if compact:
            from tracegen.format import to_c32
            r32, rop = to_c32(trace)
            return DeviceTrace(None, wo, trace.kdesc, torch.from_numpy(r32.view(np.int32)).to(device),
                               torch.from_numpy(rop).to(device))
        rec = torch.from_numpy(np.ascontiguousarray(trace.rec).view(np.int64)).to(device)
        return DeviceTrace(rec, wo, trace.kdesc)

    def record_bytes(self) -> int:
        if self.format == HR_TRACE_PACKED:
            return int(self.packed.numel())
        if self.format == HR_TRACE_POOLED:
            return self.n_rows * 288
        return self.n_rows * (160 if self.format == HR_TRACE_C32 else 256)

    def to_host(self) -> "HostTrace":
        """Pinned host copy (for hr_replay_trace_host)."""
        import torch

        def pin(x):
            h = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
            h.copy_(x)
            return h.numpy()
        wo = pin(self.warp_off).view(np.uint64)
        if self.format == HR_TRACE_PACKED:
            return HostTrace(self.kdesc, wo, packed=pin(self.packed), pack_off=pin(self.pack_off).view(np.uint64),
                             n_rows=self.n_rows)
        if self.format == HR_TRACE_C32:
            return HostTrace(self.kdesc, wo, rec32=pin(self.rec32).view(np.uint32), recop=pin(self.recop))
        return HostTrace(self.kdesc, wo, rec=pin(self.rec).view(np.uint64))

    def c(self, kernel_base: int = 0) -> HrTrace:
        t = HrTrace()
        t.n_rows = self.n_rows
        t.kdesc = self.kdesc.ctypes.data
        t.n_kernels = self.kdesc.shape[0]
        t.kernel_base = kernel_base
        t.warp_off = self.warp_off.data_ptr()
        t.n_warp_off = self.warp_off.numel()
        t.format = self.format
        t.flags = self.flags
        if self.format == HR_TRACE_C32:
            t.rec32, t.recop = self.rec32.data_ptr(), self.recop.data_ptr()
        elif self.format == HR_TRACE_POOLED:
            t.rec, t.recop = self.rec.data_ptr(), self.recop.data_ptr()
        elif self.format == HR_TRACE_PACKED:
            t.packed, t.pack_off = self.packed.data_ptr(), self.pack_off.data_ptr()
        else:
            t.rec = self.rec.data_ptr()
        return t


class HostTrace:
    """Host arrays of one trace in any format (fields as in hr_trace)."""

    def __init__(self, kdesc, warp_off, rec=None, rec32=None, recop=None, packed=None, pack_off=None,
                 n_rows: Optional[int] = None):
        self.kdesc = np.ascontiguousarray(kdesc, dtype=np.uint64)
        self.warp_off = warp_off
        self.rec, self.rec32, self.recop, self.packed, self.pack_off = rec, rec32, recop, packed, pack_off
        self.n_rows = n_rows


def host_trace_c(trace, kernel_base: int = 0) -> HrTrace:
    """HrTrace over HOST arrays (for hr_replay_trace_host); keep `trace` alive.
    `trace` has rec (U64), rec32/recop (C32) or packed/pack_off/n_rows (PACKED)
    numpy arrays, kdesc, warp_off."""
    t = HrTrace()
    t.kdesc = trace.kdesc.ctypes.data
    t.n_kernels = trace.kdesc.shape[0]
    t.kernel_base = kernel_base
    t.warp_off = trace.warp_off.ctypes.data
    t.n_warp_off = trace.warp_off.shape[0]
    if getattr(trace, "packed", None) is not None:
        t.format = HR_TRACE_PACKED
        t.n_rows = int(trace.n_rows)
        t.packed, t.pack_off = trace.packed.ctypes.data, trace.pack_off.ctypes.data
    elif getattr(trace, "rec32", None) is not None:
        t.format = HR_TRACE_C32
        t.n_rows = trace.rec32.shape[0] // 32
        t.rec32, t.recop = trace.rec32.ctypes.data, trace.recop.ctypes.data
    else:
        t.n_rows = trace.rec.shape[0] // 32
        t.rec = trace.rec.ctypes.data
    return t


def trace_extent(trace) -> Tuple[int, int]:
    """(max global word + 1, max shared words) over a host trace — for sizing shadows."""
    rec = np.asarray(trace.rec, dtype=np.uint64)
    op = rec >> np.uint64(62)
    acc = op != 3
    sp = ((rec >> np.uint64(61)) & np.uint64(1)).astype(bool)
    words = rec & np.uint64((1 << 61) - 1)
    g = words[acc & ~sp]
    gmax = int(g.max()) + 1 if g.size else 1
    smem = int(trace.kdesc[:, 3].max()) if trace.kdesc.shape[0] else 0
    return gmax, smem


class Checker:
    """One hr_ctx with a global shadow region and a shared-shadow budget."""

    def __init__(self, global_words: int, smem_words: int = 0, base_word: int = 0, device: int = 0,
                 bc_bits: int = 16, wc_bits: int = 16, ring_capacity: int = 1 << 20, options: int = 0,
                 shard: Optional[Tuple[int, int]] = None, granule_log2: int = 3, spill_capacity: int = 0):
        self.ctx = hr_init(bc_bits, wc_bits, ring_capacity, device, options, spill_capacity)
        if shard is not None:
            hr_set_shard(self.ctx, shard[0], shard[1], granule_log2)
        self.shadow_ptr = hr_shadow_alloc(self.ctx, HR_GLOBAL, base_word, max(1, global_words))
        hr_shadow_alloc(self.ctx, HR_SHARED, 0, smem_words)

    def replay(self, dtrace: DeviceTrace, stream: Optional[int] = None, kernel_base: int = 0):
        if stream is None:
            import torch
            stream = torch.cuda.current_stream().cuda_stream
        hr_replay_trace(self.ctx, dtrace.c(kernel_base), stream)

    def replay_host(self, trace, stream: Optional[int] = None, kernel_base: int = 0):
        """`trace`: numpy arrays (rec, or rec32/recop) + kdesc + warp_off in host memory."""
        if stream is None:
            import torch
            stream = torch.cuda.current_stream().cuda_stream
        self._host_ref = trace
        hr_replay_trace_host(self.ctx, host_trace_c(trace, kernel_base), stream)

    def pack(self, dtrace: DeviceTrace, stream: Optional[int] = None) -> DeviceTrace:
        """HR_TRACE_PACKED copy of a device U64 trace (hr_pack_trace)."""
        import torch
        if stream is None:
            stream = torch.cuda.current_stream().cuda_stream
        dev = dtrace.warp_off.device
        pack_off = torch.empty(dtrace.warp_off.numel(), dtype=torch.int64, device=dev)
        t = dtrace.c()
        n = hr_pack_trace(self.ctx, t, 0, 0, pack_off.data_ptr(), stream)
        out = torch.empty(n, dtype=torch.uint8, device=dev)
        hr_pack_trace(self.ctx, t, out.data_ptr(), n, pack_off.data_ptr(), stream)
        return DeviceTrace(None, dtrace.warp_off, dtrace.kdesc, packed=out, pack_off=pack_off, n_rows=dtrace.n_rows)

    def pool(self, dtrace: DeviceTrace, stream: Optional[int] = None) -> DeviceTrace:
        """HR_TRACE_POOLED copy of a device U64 / C32 trace (hr_pool_trace): this
        ctx's shard only, accesses packed 32 per row per warp epoch."""
        import torch
        if stream is None:
            stream = torch.cuda.current_stream().cuda_stream
        dev = dtrace.warp_off.device
        t = dtrace.c()
        n = hr_pool_trace(self.ctx, t, 0, 0, 0, 0, stream)
        rec = torch.empty(max(n, 1) * 32, dtype=torch.int64, device=dev)
        tag = torch.empty(max(n, 1) * 32, dtype=torch.uint8, device=dev)
        woff = torch.zeros_like(dtrace.warp_off)
        hr_pool_trace(self.ctx, t, rec.data_ptr(), tag.data_ptr(), max(n, 1), woff.data_ptr(), stream)
        out = DeviceTrace(rec[: n * 32], woff, dtrace.kdesc, recop=tag[: n * 32], pooled=True)
        out.flags = dtrace.flags
        return out

    def report(self):
        return hr_report(self.ctx)

    def report_raw(self, copy: bool = True):
        return hr_report_raw(self.ctx, copy=copy)

    def report_async(self, stream: Optional[int] = None):
        hr_report_async(self.ctx, stream)

    def collect_raw(self, copy: bool = True):
        return hr_report_collect(self.ctx, copy=copy)

    def classes(self, dtrace: "DeviceTrace", raw: np.ndarray, stream: Optional[int] = None,
                kernel_base: int = 0) -> np.ndarray:
        if stream is None:
            import torch
            stream = torch.cuda.current_stream().cuda_stream
        return hr_race_classes(self.ctx, dtrace.c(kernel_base), raw, stream)

    def reset(self):
        hr_reset_report(self.ctx)

    def close(self):
        if self.ctx:
            hr_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def check_trace(trace, device: int = 0, compact: bool = False, packed: bool = False, pooled: bool = False,
                **kw) -> Tuple[List[Race], int]:
    """Replay a host trace on the GPU and return (sorted racy set, flags).
    packed=True replays the hr_pack_trace encoding of it instead, pooled=True
    the hr_pool_trace layout."""
    gmax, smem = trace_extent(trace)
    reps = kw.pop("representatives", None)
    ck = Checker(gmax, smem, device=device, **kw)
    if reps is not None:
        hr_set_representatives(ck.ctx, *reps)
    dt = DeviceTrace.from_trace(trace, device=f"cuda:{device}", compact=compact and not packed)
    if packed:
        dt = ck.pack(dt)
    if pooled:
        dt = ck.pool(dt)
    ck.replay(dt)
    races, flags, _ = ck.report()
    ck.close()
    return races, flags
