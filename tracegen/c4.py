"""C4 workload (BASELINE.json configs[3]) — RMAT BFS levels + degree histogram
(tracegen/c4gen.c).  INPUT ONLY."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from .format import Trace

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "c4gen.c")
_LIB = os.path.join(_HERE, "libc4gen.so")
DEFAULT_SEED = 0xC4_2401


def build(force: bool = False) -> None:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=gnu99", "-fopenmp", "-shared", "-fPIC", "-o", _LIB, _SRC])


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB)
        vp, u64, u32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32
        _lib.c4_build.argtypes = [u64, u32, u32]
        _lib.c4_build.restype = vp
        _lib.c4_free.argtypes = [vp]
        _lib.c4_stats.argtypes = [vp, vp]
        _lib.c4_sizes.argtypes = [vp, ctypes.c_int, ctypes.POINTER(u64), ctypes.POINTER(u32), ctypes.POINTER(u64)]
        _lib.c4_fill.argtypes = [vp, ctypes.c_int, vp, vp, vp]
        _lib.c4_export.argtypes = [vp, vp, vp, vp]
    return _lib


class Graph:
    def __init__(self, lv: int = 24, deg: int = 16, seed: int = DEFAULT_SEED):
        self.lib = _load()
        self.h = self.lib.c4_build(seed, lv, deg)
        st = np.zeros(5, dtype=np.uint64)
        self.lib.c4_stats(self.h, st.ctypes.data)
        self.n, self.m, self.n_levels, self.reached, self.maxdeg = (int(x) for x in st)

    def trace(self, racy: bool = True) -> Trace:
        nr, nk, nw = ctypes.c_uint64(), ctypes.c_uint32(), ctypes.c_uint64()
        self.lib.c4_sizes(self.h, int(racy), ctypes.byref(nr), ctypes.byref(nk), ctypes.byref(nw))
        rec = np.empty(nr.value * 32, dtype=np.uint64)
        kd = np.zeros((nk.value, 8), dtype=np.uint64)
        wo = np.empty(nw.value, dtype=np.uint64)
        self.lib.c4_fill(self.h, int(racy), rec.ctypes.data, kd.ctypes.data, wo.ctypes.data)
        return Trace(rec, kd, wo)

    def csr(self):
        """(row_ptr uint64[n+1], col uint32[m], final BFS level int32[n], -1 = unreached)."""
        rp = np.empty(self.n + 1, dtype=np.uint64)
        col = np.empty(self.m, dtype=np.uint32)
        lvl = np.empty(self.n, dtype=np.int32)
        self.lib.c4_export(self.h, rp.ctypes.data, col.ctypes.data, lvl.ctypes.data)
        return rp, col, lvl

    def close(self):
        if self.h:
            self.lib.c4_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def total_words(lv: int) -> int:
    return (1 << lv) + 1024
