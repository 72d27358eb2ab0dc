"""CPU oracle for the split-FP16 SGEMM (arXiv 2011.11188, Appendix A).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2011_11188_b200``) never imports it, and this
package never imports the product path: they share no code.

The arithmetic lives in ``oracle.c`` (plain C, fp64, OpenMP over output rows);
this module only compiles it with gcc and marshals numpy arrays through ctypes.
Every function cites the PAPER.md passage it follows (see oracle.c and DESIGN.md
§3 for the readings R1..R9 where the paper is silent).

Pins (tests/test_oracle_*.py, marker "not gpu"): the encoder against numpy's
float32/float64 -> float16 conversion and the SPEC boundary examples; decode
against all 65536 patterns; the scale rule against its closed form; the split
against the reconstruction bound, the fp16-representable special case and the
worked example of SPEC.md:133; the split product against exact rational
arithmetic (brute force, N <= 8) and exact integer products; the dropped term
against its 2^-22 identity.  No function is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

_i64 = ctypes.c_int64
_p = ctypes.c_void_p


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with gcc (no fast-math, no FP contraction)."""
    if not force and os.path.exists(_LIB) and os.path.getmtime(_LIB) >= os.path.getmtime(_SRC):
        return _LIB
    tmp = _LIB + f".tmp{os.getpid()}"
    cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
           "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"]
    subprocess.check_call(cmd)
    os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            lib.orc_enc16.restype = ctypes.c_uint16
            lib.orc_enc16.argtypes = [ctypes.c_double]
            lib.orc_dec16.restype = ctypes.c_double
            lib.orc_dec16.argtypes = [ctypes.c_uint16]
            lib.orc_scale_exp.restype = ctypes.c_int
            lib.orc_scale_exp.argtypes = [ctypes.c_double]
            lib.orc_maxabs.restype = _i64
            lib.orc_maxabs.argtypes = [_i64, _i64, _p, _i64, _p]
            lib.orc_enc16_array.argtypes = [_i64, _p, _p]
            lib.orc_enc16_f32_array.argtypes = [_i64, _p, _p]
            lib.orc_dec16_array.argtypes = [_i64, _p, _p]
            lib.orc_split.argtypes = [_i64, _i64, _p, _i64, ctypes.c_int, _p, _p, _i64]
            lib.orc_reconstruct.argtypes = [_i64, _i64, _p, _p, _i64, ctypes.c_int, _p, _i64]
            lib.orc_gemm64.argtypes = [_i64, _i64, _i64, _p, _i64, _p, _i64, _p, _i64]
            lib.orc_split_gemm.argtypes = [_i64, _i64, _i64, _p, _p, _i64, ctypes.c_int,
                                           _p, _p, _i64, ctypes.c_int, ctypes.c_int, _p, _i64]
            lib.orc_dropped_term.argtypes = [_i64, _i64, _i64, _p, _i64, ctypes.c_int,
                                             _p, _i64, ctypes.c_int, _p, _i64]
            lib.orc_sgemm_sampled.restype = _i64
            lib.orc_sgemm_sampled.argtypes = [_i64, _i64, _i64, _p, _i64, _p, _i64,
                                              _i64, _p, _i64, _p, ctypes.c_int, _p, _p, _p]
            lib.orc_encbf16.restype = ctypes.c_uint16
            lib.orc_encbf16.argtypes = [ctypes.c_double]
            lib.orc_decbf16.restype = ctypes.c_double
            lib.orc_decbf16.argtypes = [ctypes.c_uint16]
            lib.orc_encbf16_array.argtypes = [_i64, _p, _p]
            lib.orc_split_bf16x3.argtypes = [_i64, _i64, _p, _i64, _p, _p, _p, _i64]
            lib.orc_gemm_bf16x3.argtypes = [_i64, _i64, _i64, _p, _p, _p, _i64, _p, _p, _p, _i64, _p, _i64]
            lib.orc_num_threads.restype = ctypes.c_int
            lib.orc_set_num_threads.argtypes = [ctypes.c_int]
            _lib = lib
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


# ---------------------------------------------------------------- binary16 ---

def enc16(x) -> np.ndarray:
    """RNE fp64/fp32 -> binary16 bit patterns (uint16), bit by bit."""
    x = np.asarray(x)
    if x.dtype == np.float32:
        xf = np.ascontiguousarray(x)
        out = np.empty(xf.shape, np.uint16)
        _load().orc_enc16_f32_array(xf.size, _ptr(xf), _ptr(out))
        return out
    xd = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty(xd.shape, np.uint16)
    _load().orc_enc16_array(xd.size, _ptr(xd), _ptr(out))
    return out


def dec16(h) -> np.ndarray:
    """binary16 bit patterns -> exact fp64 values."""
    h = np.ascontiguousarray(h, dtype=np.uint16)
    out = np.empty(h.shape, np.float64)
    _load().orc_dec16_array(h.size, _ptr(h), _ptr(out))
    return out


# ------------------------------------------------------------------- scale ---

def scale_exp(m: float) -> int:
    """Reading R1: s = 0 if m == 0 else max(floor(log2 m) - 14, -127)."""
    return int(_load().orc_scale_exp(float(m)))


def maxabs(X) -> tuple[float, int]:
    """(max |x| over finite entries, first non-finite linear index or -1)."""
    X = _f32(X)
    rows, cols = X.shape
    out = np.zeros(1, np.float64)
    bad = _load().orc_maxabs(rows, cols, _ptr(X), cols, _ptr(out))
    return float(out[0]), int(bad)


# ------------------------------------------------------------------- split ---

def split(X, s: int | None = None):
    """Eq. A_1 split of a row-major fp32 matrix -> (hi, lo, s) with uint16 planes.

    ``s`` defaults to the per-matrix scale exponent of X (reading R1); pass the
    global exponent when X is a shard or a sample of a larger matrix.
    """
    X = _f32(X)
    if X.ndim != 2:
        raise ValueError("split expects a 2-D matrix")
    rows, cols = X.shape
    if s is None:
        m, bad = maxabs(X)
        if bad >= 0:
            raise ValueError(f"non-finite entry at linear index {bad}")
        s = scale_exp(m)
    hi = np.empty((rows, cols), np.uint16)
    lo = np.empty((rows, cols), np.uint16)
    _load().orc_split(rows, cols, _ptr(X), cols, int(s), _ptr(hi), _ptr(lo), cols)
    return hi, lo, int(s)


def reconstruct(hi, lo, s: int) -> np.ndarray:
    """a1*A1 + a2*A2 in fp64, a1 = 2^s, a2 = 2^(s-11)."""
    hi = np.ascontiguousarray(hi, np.uint16)
    lo = np.ascontiguousarray(lo, np.uint16)
    rows, cols = hi.shape
    out = np.empty((rows, cols), np.float64)
    _load().orc_reconstruct(rows, cols, _ptr(hi), _ptr(lo), cols, int(s), _ptr(out), cols)
    return out


# -------------------------------------------------------------------- gemm ---

def gemm64(A, B) -> np.ndarray:
    """C64 = A*B in fp64 (exact products, fp64 sums)."""
    A = _f32(A)
    B = _f32(B)
    M, K = A.shape
    K2, N = B.shape
    if K != K2:
        raise ValueError("inner dimensions differ")
    C = np.empty((M, N), np.float64)
    _load().orc_gemm64(M, N, K, _ptr(A), K, _ptr(B), N, _ptr(C), N)
    return C


def split_gemm(A1, A2, sA: int, B1, B2, sB: int, terms: int = 3) -> np.ndarray:
    """Eq. A_2 product of split planes (A planes M x K, B planes K x N), fp64."""
    if terms not in (1, 3, 4):
        raise ValueError("terms must be 1, 3 or 4")
    A1 = np.ascontiguousarray(A1, np.uint16)
    A2 = np.ascontiguousarray(A2, np.uint16)
    B1 = np.ascontiguousarray(B1, np.uint16)
    B2 = np.ascontiguousarray(B2, np.uint16)
    M, K = A1.shape
    K2, N = B1.shape
    if K != K2 or A2.shape != A1.shape or B2.shape != B1.shape:
        raise ValueError("plane shapes differ")
    C = np.empty((M, N), np.float64)
    _load().orc_split_gemm(M, N, K, _ptr(A1), _ptr(A2), K, int(sA),
                           _ptr(B1), _ptr(B2), N, int(sB), int(terms), _ptr(C), N)
    return C


def dropped_term(A2, sA: int, B2, sB: int) -> np.ndarray:
    """2^(sA+sB-22) * A2*B2 in fp64."""
    A2 = np.ascontiguousarray(A2, np.uint16)
    B2 = np.ascontiguousarray(B2, np.uint16)
    M, K = A2.shape
    _, N = B2.shape
    C = np.empty((M, N), np.float64)
    _load().orc_dropped_term(M, N, K, _ptr(A2), K, int(sA), _ptr(B2), N, int(sB), _ptr(C), N)
    return C


def sgemm(A, B, terms: int = 3) -> np.ndarray:
    """End-to-end emulated C = A*B: per-matrix scales, split, Eq. A_2 in fp64."""
    A1, A2, sA = split(A)
    B1, B2, sB = split(B)
    return split_gemm(A1, A2, sA, B1, B2, sB, terms)


def sgemm_sampled(A, B, rows, cols, terms: int = 3):
    """Emulated C[rows][:, cols] with scales taken from the whole A and B.

    Returns (C_sample fp64 of shape (len(rows), len(cols)), sA, sB).
    """
    A = _f32(A)
    B = _f32(B)
    M, K = A.shape
    _, N = B.shape
    rows = np.ascontiguousarray(rows, np.int64)
    cols = np.ascontiguousarray(cols, np.int64)
    out = np.empty((rows.size, cols.size), np.float64)
    sA = np.zeros(1, np.int32)
    sB = np.zeros(1, np.int32)
    bad = _load().orc_sgemm_sampled(M, N, K, _ptr(A), K, _ptr(B), N, rows.size, _ptr(rows),
                                    cols.size, _ptr(cols), int(terms), _ptr(out),
                                    _ptr(sA), _ptr(sB))
    if bad >= 0:
        raise ValueError(f"non-finite entry at index {bad}")
    return out, int(sA[0]), int(sB[0])


# ------------------------------------------------------- bf16 x 3 (NEXT #4) ---

def encbf16(x) -> np.ndarray:
    """RNE fp64 -> bfloat16 bit patterns (uint16), bit by bit."""
    xd = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty(xd.shape, np.uint16)
    _load().orc_encbf16_array(xd.size, _ptr(xd), _ptr(out))
    return out


def decbf16(h) -> np.ndarray:
    """bfloat16 bit patterns -> exact fp64 values (bf16 is the top half of binary32)."""
    h = np.ascontiguousarray(h, dtype=np.uint16)
    with np.errstate(invalid="ignore"):     # signalling-NaN patterns
        return (h.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def split_bf16x3(X):
    """(X1, X2, X3) bfloat16 planes (uint16) of a row-major fp32 matrix (no scale)."""
    X = _f32(X)
    rows, cols = X.shape
    p = [np.empty((rows, cols), np.uint16) for _ in range(3)]
    _load().orc_split_bf16x3(rows, cols, _ptr(X), cols, _ptr(p[0]), _ptr(p[1]), _ptr(p[2]), cols)
    return tuple(p)


def gemm_bf16x3_planes(X, Y):
    """6-term product of bf16x3 planes X = (X1,X2,X3) (M x K), Y = (Y1,Y2,Y3) (K x N), fp64."""
    X = [np.ascontiguousarray(v, np.uint16) for v in X]
    Y = [np.ascontiguousarray(v, np.uint16) for v in Y]
    M, K = X[0].shape
    _, N = Y[0].shape
    C = np.empty((M, N), np.float64)
    _load().orc_gemm_bf16x3(M, N, K, _ptr(X[0]), _ptr(X[1]), _ptr(X[2]), K, _ptr(Y[0]), _ptr(Y[1]),
                            _ptr(Y[2]), N, _ptr(C), N)
    return C


def sgemm_bf16x3(A, B):
    return gemm_bf16x3_planes(split_bf16x3(A), split_bf16x3(B))


def num_threads() -> int:
    return int(_load().orc_num_threads())


def set_num_threads(n: int) -> None:
    _load().orc_set_num_threads(int(n))
