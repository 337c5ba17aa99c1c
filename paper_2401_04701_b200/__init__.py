"""B200-native HiRace per-access race check (arXiv 2401.04701).

The product path is libhirace.so (csrc/, sm_100a) behind the C ABI in
include/hr.h; ``hirace`` is its ctypes binding.  Importing this package does
not touch CUDA; ``hirace.load()`` raises if the library is missing.
"""
__all__ = ["hirace", "build"]
