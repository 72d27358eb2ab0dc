"""B200-native split-FP16 SGEMM (arXiv 2011.11188, Appendix A).

C = A*B for FP32 A, B emulated by three FP16 tcgen05 GEMMs:
A ~= a1*A1 + a2*A2, B ~= b1*B1 + b2*B2 (a2 = 2^-11 a1), C ~= a1b1 (A1B1 + 2^-11 (A1B2 + A2B1)).
The product path is libsplit3.so (csrc/, include/split3.h); this package is its binding
(split3.py) and the multi-GPU 2-D tile driver (dist.py).
"""
from .split3 import (CHECK_FINITE, FOUR_TERM, ONE_TERM, THREE_TERM, Handle, NotFiniteError, Planes,
                     Split3Error, handle, load, plane_ld, sgemm)

__all__ = ["sgemm", "handle", "Handle", "Planes", "load", "plane_ld", "Split3Error", "NotFiniteError",
           "THREE_TERM", "FOUR_TERM", "ONE_TERM", "CHECK_FINITE"]
