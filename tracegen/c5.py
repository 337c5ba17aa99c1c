"""C5 workload (BASELINE.json configs[4]) — CPU and GPU builds of the same
counter-based generator (c5gen.h).  INPUT ONLY."""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import List, Tuple

import numpy as np

from .format import Trace

_HERE = os.path.dirname(os.path.abspath(__file__))
_CPU_LIB = os.path.join(_HERE, "libc5gen_cpu.so")
_GPU_LIB = os.path.join(_HERE, "libc5gen_cuda.so")
_HDR = os.path.join(_HERE, "c5gen.h")

WARPS, LANES, ACC, ROWS = 8, 32, 256, 264
DEFAULT_SEED = 0x5EED_C5


class Params(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("lb", ctypes.c_uint32)]


def _stale(lib, src):
    return (not os.path.exists(lib) or os.path.getmtime(lib) < os.path.getmtime(src)
            or os.path.getmtime(lib) < os.path.getmtime(_HDR))


def build(force: bool = False) -> None:
    src = os.path.join(_HERE, "c5gen.c")
    if force or _stale(_CPU_LIB, src):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-shared", "-fPIC", "-o", _CPU_LIB, src])
    src = os.path.join(_HERE, "c5gen.cu")
    if force or _stale(_GPU_LIB, src):
        nvcc = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
        subprocess.check_call([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                               "-Xcompiler", "-fPIC", "-o", _GPU_LIB, src])


_cpu = None
_gpu = None


def _cpu_lib():
    global _cpu
    if _cpu is None:
        build()
        _cpu = ctypes.CDLL(_CPU_LIB)
        P = ctypes.POINTER
        _cpu.c5_warp_rows.argtypes = [P(Params), ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                      ctypes.c_uint64]
        _cpu.c5_warp_rows.restype = ctypes.c_uint64
        _cpu.c5_gen_cpu.argtypes = [P(Params), ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64,
                                    ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p]
        _cpu.c5_planted.argtypes = [P(Params), ctypes.c_void_p, ctypes.c_void_p]
        _cpu.c5_record_at.argtypes = [P(Params), ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32]
        _cpu.c5_record_at.restype = ctypes.c_uint64
    return _cpu


def _gpu_lib():
    global _gpu
    if _gpu is None:
        build()
        _gpu = ctypes.CDLL(_GPU_LIB)
        _gpu.c5_gen_gpu.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                    ctypes.c_uint32, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        _gpu.c5_gen_gpu.restype = ctypes.c_int
    return _gpu


def _log2(n: int) -> int:
    assert n >= 1 and n & (n - 1) == 0, "shard count must be a power of two"
    return n.bit_length() - 1


def total_words(lb: int) -> int:
    return 1 << (lb + 16)


def n_accesses(lb: int) -> int:
    return (1 << lb) * 256 * ACC


def kdesc(lb: int) -> np.ndarray:
    return np.array([[1 << lb, WARPS, LANES, 0, 0, 0, 0, 0]], dtype=np.uint64)


def cpu_trace(lb: int, seed: int = DEFAULT_SEED, rank: int = 0, nshard: int = 1, granule_log2: int = 3) -> Trace:
    """The (shard of the) C5 trace as host arrays."""
    lib = _cpu_lib()
    p = Params(seed, lb)
    nw = (1 << lb) * WARPS
    l2 = _log2(nshard)
    rows = np.array([lib.c5_warp_rows(ctypes.byref(p), rank, l2, granule_log2, w) for w in range(nw)],
                    dtype=np.uint64)
    off = np.zeros(nw + 1, dtype=np.uint64)
    off[1:] = np.cumsum(rows)
    rec = np.empty(int(off[-1]) * 32, dtype=np.uint64)
    lib.c5_gen_cpu(ctypes.byref(p), rank, l2, granule_log2, 0, nw, off.ctypes.data, rec.ctypes.data)
    return Trace(rec, kdesc(lb), off)


def planted(lb: int, seed: int = DEFAULT_SEED) -> List[Tuple[int, int]]:
    """The closed-form racy set: [(word, scope)] sorted by word."""
    lib = _cpu_lib()
    p = Params(seed, lb)
    n = 1 << lb
    w = np.empty(n, dtype=np.uint64)
    s = np.empty(n, dtype=np.uint8)
    lib.c5_planted(ctypes.byref(p), w.ctypes.data, s.ctypes.data)
    return sorted(zip((int(x) for x in w), (int(x) for x in s)))


def _gpu_offsets(lib, lb, seed, rank, l2, g2, device, stream):
    import torch
    nw = (1 << lb) * WARPS
    if l2 == 0:
        return torch.arange(nw + 1, dtype=torch.int64, device=device) * ROWS
    rows = torch.empty(nw, dtype=torch.int64, device=device)
    rc = lib.c5_gen_gpu(seed, lb, rank, l2, g2, 0, rows.data_ptr(), None, None, None, None, stream)
    assert rc == 0, rc
    off = torch.zeros(nw + 1, dtype=torch.int64, device=device)
    off[1:] = torch.cumsum(rows, 0)
    return off


def gpu_trace(lb: int, seed: int = DEFAULT_SEED, rank: int = 0, nshard: int = 1, device: str = "cuda",
              granule_log2: int = 3):
    """Generate the (shard of the) trace directly in HBM, u64 records.
    Returns (rec int64 tensor, warp_off int64 tensor, kdesc numpy)."""
    import torch
    lib = _gpu_lib()
    stream = torch.cuda.current_stream().cuda_stream
    off = _gpu_offsets(lib, lb, seed, rank, _log2(nshard), granule_log2, device, stream)
    n_rows = int(off[-1].item())
    rec = torch.empty(n_rows * 32, dtype=torch.int64, device=device)
    rc = lib.c5_gen_gpu(seed, lb, rank, _log2(nshard), granule_log2, 1, None, off.data_ptr(), rec.data_ptr(),
                        None, None, stream)
    assert rc == 0, rc
    return rec, off, kdesc(lb)


def gpu_trace_c32(lb: int, seed: int = DEFAULT_SEED, rank: int = 0, nshard: int = 1, device: str = "cuda",
                  granule_log2: int = 3):
    """Same trace in the HR_TRACE_C32 encoding (160 B per row).  Returns
    (rec32 int32, recop uint8, warp_off int64) tensors and kdesc."""
    import torch
    lib = _gpu_lib()
    stream = torch.cuda.current_stream().cuda_stream
    off = _gpu_offsets(lib, lb, seed, rank, _log2(nshard), granule_log2, device, stream)
    n_rows = int(off[-1].item())
    rec32 = torch.empty(n_rows * 32, dtype=torch.int32, device=device)
    recop = torch.empty(n_rows * 32, dtype=torch.uint8, device=device)
    rc = lib.c5_gen_gpu(seed, lb, rank, _log2(nshard), granule_log2, 1, None, off.data_ptr(), None,
                        rec32.data_ptr(), recop.data_ptr(), stream)
    assert rc == 0, rc
    return rec32, recop, off, kdesc(lb)
