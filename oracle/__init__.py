"""CPU oracle for HiRace's racy-address set — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  It
shares no code with the CUDA path (``paper_2401_04701_b200``) and never
imports it.

* ``check(trace)``       — hr_oracle.c: the plain happens-before race definition
                           (§II-A), pairwise or bucketed;
                           racy addresses, their scope and their race classes.
* ``vclock``             — vector-clock detector along explicit interleavings
                           and schedule enumeration,
                           pure Python, tiny traces only.

Parity status: every function here is pinned by tests/test_oracle_pins.py
(paper listings, closed forms, vector clocks over all interleavings,
pairwise == bucketed).  No function is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import List, NamedTuple, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hr_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

PAIRWISE, BUCKETED = 0, 1
F_CLOCK_OVERFLOW, F_MODEL_VIOLATION, F_BARRIER_DIVERGENCE = 1, 4, 8
SCOPE_BLOCK, SCOPE_GRID = 1, 2
GLOBAL_BLOCK = 0xFFFFFFFF


class Race(NamedTuple):
    kernel: int
    space: int
    block: int
    word: int
    scope: int


class _RaceC(ctypes.Structure):
    _fields_ = [("word", ctypes.c_uint64), ("kernel", ctypes.c_uint32), ("block", ctypes.c_uint32),
                ("space", ctypes.c_uint8), ("scope", ctypes.c_uint8), ("classes", ctypes.c_uint8),
                ("pad", ctypes.c_uint8 * 5)]

CLASS_WW, CLASS_RW, CLASS_AW, CLASS_AR = 1, 2, 4, 8


def build(force: bool = False) -> str:
    """Compile hr_oracle.c with gcc (plain C, -O2)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.POINTER
        _lib.hro_check.argtypes = [P(ctypes.c_uint64), P(ctypes.c_uint64), ctypes.c_uint64,
                                   P(ctypes.c_uint64), ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32,
                                   P(_RaceC), ctypes.c_uint64, P(ctypes.c_uint64), P(ctypes.c_uint32),
                                   P(ctypes.c_uint64)]
        _lib.hro_check.restype = ctypes.c_int
        _lib.hro_sizeof_race.restype = ctypes.c_uint64
        assert _lib.hro_sizeof_race() == ctypes.sizeof(_RaceC)
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))


class Result(NamedTuple):
    races: List[Race]
    flags: int
    n_accesses: int
    classes: List[int] = []      # per race: bit0 W-W, bit1 R-W, bit2 A-W, bit3 A-R


def check(trace, mode: int = BUCKETED, bc_bits: int = 16, wc_bits: int = 16) -> Result:
    """Sorted racy set of ``trace`` (a tracegen.Trace or any object with
    ``rec``, ``kdesc``, ``warp_off`` uint64 arrays)."""
    lib = _load()
    rec = np.ascontiguousarray(trace.rec, dtype=np.uint64)
    kd = np.ascontiguousarray(trace.kdesc, dtype=np.uint64)
    wo = np.ascontiguousarray(trace.warp_off, dtype=np.uint64)
    cap = 1024
    while True:
        out = (_RaceC * cap)()
        n = ctypes.c_uint64(0)
        fl = ctypes.c_uint32(0)
        na = ctypes.c_uint64(0)
        rc = lib.hro_check(_ptr(rec), _ptr(kd), kd.shape[0], _ptr(wo), mode,
                           (1 << bc_bits) - 1, (1 << wc_bits) - 1, out, cap,
                           ctypes.byref(n), ctypes.byref(fl), ctypes.byref(na))
        if rc == -3:
            cap = int(n.value) + 16
            continue
        if rc != 0:
            raise RuntimeError(f"hro_check failed: {rc}")
        races = [Race(int(r.kernel), int(r.space), int(r.block), int(r.word), int(r.scope))
                 for r in out[: n.value]]
        return Result(races, int(fl.value), int(na.value), [int(r.classes) for r in out[: n.value]])


def racy_words(result: Result) -> List[int]:
    return [r.word for r in result.races]
