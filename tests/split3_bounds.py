"""Per-element error bound of the split GEMM against the oracle; shared by the
GPU parity tests.  Test infrastructure only."""
import numpy as np


def _elementwise_bound(orc, A, B, terms, slices=16):
    """Per-element bound on |C_gpu - C_split| (C_split: the oracle's fp64 Eq. A_2), from the
    measured accumulator semantics (DESIGN.md §3 R9): one kind::f16 MMA sums 16 exact products
    into the FP32 accumulator with truncation, losing < 1 ulp of the largest addend per addend
    (<= 18 u M per MMA, u = 2^-23, M <= the partial sum of |products|); D_hi is promoted with
    round-to-nearest every 8 MMAs (library default), D_mid (D_lo) accumulate over the whole K;
    split-K slices are added with RN; the epilogue fma rounds once, the 2^(sA+sB) scale is exact.
        |err_ij| <= 2^(sA+sB) [ (144 u + (K/128 + 1 + slices) u/2) S_hi
                               + 2^-11 (18 ceil(K/16) + 1) u S_mid + 2^-22 (18 ceil(K/16) + 1) u S_lo ]
                    + u/2 |C_split|
    with S_hi = |A1| |B1|, S_mid = |A1||B2| + |A2||B1|, S_lo = |A2||B2| (decoded planes)."""
    K = A.shape[1]
    a1, a2, sA = orc.split(A)
    b1, b2, sB = orc.split(B)
    A1, A2 = np.abs(orc.dec16(a1)), np.abs(orc.dec16(a2))
    B1, B2 = np.abs(orc.dec16(b1)), np.abs(orc.dec16(b2))
    u = 2.0 ** -23
    nk = -(-K // 16)
    bnd = (144 * u + (K / 128 + 1 + slices) * u / 2) * (A1 @ B1)
    if terms != 1:
        bnd += 2.0 ** -11 * (18 * nk + 1) * u * (A1 @ B2 + A2 @ B1)
    if terms == 4:
        bnd += 2.0 ** -22 * (18 * nk + 1) * u * (A2 @ B2)
    return np.ldexp(bnd, sA + sB)


def _elementwise_bound_fold(orc, A, B, terms, slices=16):
    """The same bound for the folded accumulator (split3_set_fold): per 64-wide
    k-block ONE accumulator T takes [4 MMAs of A2*B2 (4-term)], then 8 MMAs of A1*B2 + A2*B1
    entered with T <- P + 2^-11 T (exact power-of-two scaling), then 4 MMAs of A1*B1 likewise, and
    is promoted (RN) every k-block.  Each MMA loses < 18 u M (M <= the partial sum of |products|
    in T's units, lower groups included), so with S = S_hi + 2^-11 S_mid + 2^-22 S_lo:
        |err_ij| <= 2^(sA+sB) [ (72 u + (K/64 + slices) u/2) S + 2^-11 144 u (S_mid + 2^-11 S_lo)
                               + 2^-22 72 u S_lo ] + u/2 |C_split|"""
    K = A.shape[1]
    a1, a2, sA = orc.split(A)
    b1, b2, sB = orc.split(B)
    A1, A2 = np.abs(orc.dec16(a1)), np.abs(orc.dec16(a2))
    B1, B2 = np.abs(orc.dec16(b1)), np.abs(orc.dec16(b2))
    u = 2.0 ** -23
    nkb = -(-K // 64)
    s_hi = A1 @ B1
    s_mid = A1 @ B2 + A2 @ B1
    s_lo = A2 @ B2 if terms == 4 else np.zeros_like(s_hi)
    S = s_hi + 2.0 ** -11 * s_mid + 2.0 ** -22 * s_lo
    bnd = (72 * u + (nkb + slices) * u / 2) * S + 2.0 ** -11 * 144 * u * (s_mid + 2.0 ** -11 * s_lo) \
        + 2.0 ** -22 * 72 * u * s_lo
    return np.ldexp(bnd, sA + sB)


def _assert_elementwise(orc, C, Cs, A, B, terms, fold=None):
    """fold: the folded accumulator's bound (None: the library default — folded for 4-term calls of
    at least 8192^3 multiply-adds)"""
    if fold is None:
        fold = terms == 4 and A.shape[0] * B.shape[1] * A.shape[1] >= 2 ** 39
    bound = (_elementwise_bound_fold(orc, A, B, terms) if fold else _elementwise_bound(orc, A, B, terms)) \
        + 2.0 ** -24 * np.abs(Cs)
    err = np.abs(C.astype(np.float64) - Cs)
    bad = np.argwhere(err > bound)
    assert bad.size == 0, (bad[:5].tolist(), err[tuple(bad[0])], bound[tuple(bad[0])])
    return float(np.max(err / np.maximum(bound, 1e-300)))
