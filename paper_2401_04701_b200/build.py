"""Build the sm_100a CUDA library in-tree (nvcc -shared, no JIT cache)."""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libhirace.so")
LIB_FUZZ = os.path.join(PKG, "libhirace_fuzz.so")   # -DHR_FUZZ schedule-fuzzing variant (tests only)
SOURCES = [os.path.join(CSRC, "hr_host.cu"), os.path.join(CSRC, "hr_online.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("hr_replay.cuh", "hr_records.cuh", "hr_fh.cuh", "hr_classes.cuh", "hr_pack.cuh", "hr_compact.cuh", "hr_streams.cuh", "hr_binned.cuh", "hr_bserial.cuh", "fsm_table.inc",
                                            "fsm_classes.inc")] + \
    [os.path.join(INCLUDE, f) for f in ("hr.h", "hr_device.cuh", "hr_bench.h", "hr_array.cuh")]

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-shared", "-Xcompiler", "-fPIC", "-Xptxas", "-v"]


def nvcc() -> str:
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, extra=None, verbose: bool = False, lib: str = LIB) -> str:
    if lib == LIB_FUZZ:
        extra = ["-DHR_FUZZ"] + (extra or [])
    if force or stale(lib, DEPS):
        cmd = [nvcc()] + NVCC_FLAGS + (extra or []) + ["-I", INCLUDE, "-I", CSRC, "-o", lib] + SOURCES
        out = subprocess.run(cmd, capture_output=True, text=True)
        if out.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + out.stdout + out.stderr)
        if verbose:
            print(out.stderr)
    return lib


def build_fuzz(force: bool = False) -> str:
    return build(force=force, lib=LIB_FUZZ)


if __name__ == "__main__":
    print(build(force=True, verbose=True))
