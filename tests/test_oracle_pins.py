"""Pins for the CPU oracle (oracle/): each check compares the oracle with
something other than itself — numpy's independent binary16 conversion, exact
rational arithmetic, exact integer products, closed forms and the worked
example of SPEC.md:133 — chosen so that a dropped term, a wrong sign or index,
or a transposed operand in oracle.c fails at least one of them.
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from workloads import numpy_matrix

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _read_table(name):
    rows = []
    for line in open(os.path.join(GOLDEN, name)):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        rows.append(line.split()[:2])
    return rows


def _parse(v):
    if v in ("inf", "-inf", "nan"):
        return float(v)
    return float.fromhex(v)


# ------------------------------------------------------------- encode ------

def test_encode_golden(orc):
    """SPEC.md:43-45 boundary cases + binary16 format definition (golden file)."""
    for v, bits in _read_table("encode_cases.txt"):
        x = _parse(v)
        got = int(orc.enc16(np.array([x]))[0])
        assert got == int(bits, 16), (v, hex(got), bits)
        if math.isnan(x) or float(np.float32(x)) == x:
            got32 = int(orc.enc16(np.array([x], np.float32))[0])
            assert got32 == int(bits, 16), (v, hex(got32), bits)


def _numpy_half_bits(x):
    return np.asarray(x).astype(np.float16).view(np.uint16)


def test_encode_vs_numpy_fp32_strided(orc):
    """Every 97th fp32 bit pattern (44M patterns, all exponents/signs) vs numpy."""
    step = 97
    for start in range(0, 1 << 32, 1 << 28):
        bits = np.arange(start, min(start + (1 << 28), 1 << 32), step, dtype=np.uint64).astype(np.uint32)
        x = bits.view(np.float32)
        ref = _numpy_half_bits(x)
        got = orc.enc16(x)
        nan = np.isnan(x)
        assert np.array_equal(got[~nan], ref[~nan])
        assert np.all(got[nan] == 0x7E00)


def test_encode_vs_numpy_rounding_boundaries(orc):
    """All fp32 patterns whose low 13 bits sit at/around the fp16 rounding point.

    For every sign, every exponent in the fp16-relevant range (2^-27 .. 2^16)
    and every value of the upper 10 mantissa bits, the low 13 bits take the
    values {0, 1, 0xFFF, 0x1000 (tie), 0x1001, 0x1FFF}.
    """
    exps = np.arange(127 - 27, 127 + 17, dtype=np.uint32)
    hi = np.arange(1 << 10, dtype=np.uint32)
    lows = np.array([0, 1, 0xFFF, 0x1000, 0x1001, 0x1FFF], dtype=np.uint32)
    for sign in (0, 1):
        b = (np.uint32(sign) << 31) | (exps[:, None, None] << 23) | (hi[None, :, None] << 13) | lows[None, None, :]
        x = b.ravel().view(np.float32)
        assert np.array_equal(orc.enc16(x), _numpy_half_bits(x))
    # subnormal-half region in fine steps: every fp32 in [2^-26, 2^-14) with low 8 bits in a set
    for e in range(127 - 26, 127 - 14):
        m = np.arange(0, 1 << 23, 251, dtype=np.uint32)
        x = ((np.uint32(e) << 23) | m).view(np.float32)
        assert np.array_equal(orc.enc16(x), _numpy_half_bits(x))


def test_encode_fp64_vs_numpy(orc):
    """fp64 inputs (the oracle's internal precision) vs numpy's double->half."""
    rng = np.random.Generator(np.random.PCG64(7))
    e = rng.integers(-30, 18, size=2_000_000)
    m = rng.random(2_000_000) + 1.0
    x = np.ldexp(m, e) * np.where(rng.random(2_000_000) < 0.5, -1.0, 1.0)
    # exact ties and near-ties in the normal and subnormal half ranges
    q = rng.integers(0, 2048, size=200_000).astype(np.float64)
    ex = rng.integers(-24, 6, size=200_000)
    ties = np.ldexp(q + 0.5, ex)
    near = np.concatenate([ties, np.nextafter(ties, 0), np.nextafter(ties, np.inf)])
    x = np.concatenate([x, near, -near])
    assert np.array_equal(orc.enc16(x), _numpy_half_bits(x))


@pytest.mark.slow
@pytest.mark.skipif(not os.environ.get("SPLIT3_SLOW"), reason="set SPLIT3_SLOW=1 (minutes)")
def test_encode_vs_numpy_fp32_exhaustive(orc):
    """All 2^32 fp32 patterns (minutes; run with -m slow)."""
    for start in range(0, 1 << 32, 1 << 26):
        bits = np.arange(start, start + (1 << 26), dtype=np.uint64).astype(np.uint32)
        x = bits.view(np.float32)
        ref = _numpy_half_bits(x)
        got = orc.enc16(x)
        nan = np.isnan(x)
        assert np.array_equal(got[~nan], ref[~nan])


# ------------------------------------------------------------- decode ------

def test_decode_all_patterns(orc):
    h = np.arange(1 << 16, dtype=np.uint32).astype(np.uint16)
    ref = h.view(np.float16).astype(np.float64)
    got = orc.dec16(h)
    nan = np.isnan(ref)
    assert np.array_equal(got[~nan], ref[~nan])
    assert np.all(np.isnan(got[nan]))
    # roundtrip enc(dec(h)) == h for every non-NaN pattern
    assert np.array_equal(orc.enc16(got[~nan]), h[~nan])
    assert orc.dec16(np.array([1], np.uint16))[0] == 2.0 ** -24
    assert orc.dec16(np.array([0x7C00], np.uint16))[0] == np.inf


# -------------------------------------------------------------- scale ------

@pytest.mark.parametrize("m,s", [
    (0.0, 0), (1.0, -14), (0.999, -15), (0.5, -15), (2.0, -13), (3.9, -13),
    (65504.0, 1), (2.0 ** -113, -127), (2.0 ** -112, -126), (2.0 ** -120, -127),
    (2.0 ** -149, -127), (float(np.finfo(np.float32).max), 113), (1.0 + 2 ** -12, -14),
])
def test_scale_closed_form(orc, m, s):
    """Reading R1: s = max(floor(log2 m) - 14, -127), s(0) = 0."""
    assert orc.scale_exp(m) == s


def test_scale_puts_max_in_top_binades(orc):
    rng = np.random.Generator(np.random.PCG64(3))
    for m in np.ldexp(rng.random(2000) + 1.0, rng.integers(-100, 120, 2000)):
        s = orc.scale_exp(m)
        assert 2.0 ** 14 <= m * 2.0 ** -s < 2.0 ** 15


def test_maxabs_skips_nonfinite(orc):
    X = np.array([[1.0, -3.0], [np.inf, 2.0]], np.float32)
    m, bad = orc.maxabs(X)
    assert m == 3.0 and bad == 2
    X = np.array([[np.nan, -0.5]], np.float32)
    m, bad = orc.maxabs(X)
    assert m == 0.5 and bad == 0


# -------------------------------------------------------------- split ------

def test_worked_example(orc):
    """[[1+2^-12]] — golden file."""
    g = dict(_read_table("worked_example.txt"))
    x = np.array([[_parse(g["x"])]], np.float32)
    hi, lo, s = orc.split(x)
    assert s == int(g["s"])
    assert int(hi[0, 0]) == int(g["A1"], 16) and int(lo[0, 0]) == int(g["A2"], 16)
    assert orc.reconstruct(hi, lo, s)[0, 0] == float(x[0, 0])
    c3 = orc.split_gemm(hi, lo, s, hi, lo, s, terms=3)[0, 0]
    c4 = orc.split_gemm(hi, lo, s, hi, lo, s, terms=4)[0, 0]
    assert c3 == _parse(g["C3"])
    assert c4 == _parse(g["C4"])
    assert float(np.float32(c4)) == _parse(g["C3"])   # the 2^-24 term vanishes in fp32
    assert orc.dropped_term(lo, s, lo, s)[0, 0] == _parse(g["dropped"])


@pytest.mark.parametrize("kind,scale", [("uniform", 1.0), ("uniform", 2.0 ** -20), ("uniform", 2.0 ** 14),
                                        ("loguni", 1.0), ("glorot", 1.0), ("int2", 1.0)])
def test_split_reconstruction_bound(orc, kind, scale):
    """|x - a1 A1 - a2 A2| <= 2^-22 |x| + 2^(s-36) (two RN16 roundings; DESIGN.md §3 R3)."""
    X = (numpy_matrix(kind, 96, 80, seed=11) * np.float32(scale)).astype(np.float32)
    hi, lo, s = orc.split(X)
    rec = orc.reconstruct(hi, lo, s)
    x = X.astype(np.float64)
    err = np.abs(x - rec)
    assert np.all(err <= 2.0 ** -22 * np.abs(x) + 2.0 ** (s - 36))
    # A1 alone carries the leading ~3 decimal digits: rel err <= 2^-11
    a1 = np.ldexp(orc.dec16(hi), s)
    normal = np.abs(a1) >= 2.0 ** (s - 14)
    assert np.all(np.abs(x - a1)[normal] <= 2.0 ** -11 * np.abs(x)[normal])
    # no overflow: planes finite, |A1| < 2^15, |A2| <= |A1| where A1 is normal
    d1, d2 = orc.dec16(hi), orc.dec16(lo)
    assert np.all(np.isfinite(d1)) and np.all(np.isfinite(d2))
    assert np.all(np.abs(d1) <= 2.0 ** 15)
    assert np.all(np.abs(d2)[np.abs(d1) >= 2 ** -14] <= np.abs(d1)[np.abs(d1) >= 2 ** -14])


def test_split_fp16_representable_has_zero_residual(orc):
    """x fp16-representable with max|x| < 2^15 => A2 == 0 exactly, A1 = x * 2^-s."""
    X = numpy_matrix("fp16", 64, 64, seed=5)
    hi, lo, s = orc.split(X)
    assert np.all(lo & 0x7FFF == 0)
    assert np.array_equal(np.ldexp(orc.dec16(hi), s), X.astype(np.float64))


def test_split_zero_matrix(orc):
    hi, lo, s = orc.split(np.zeros((3, 5), np.float32))
    assert s == 0 and np.all(hi == 0) and np.all(lo == 0)


def test_split_uses_given_global_scale(orc):
    X = numpy_matrix("uniform", 8, 8, seed=1)
    hi, lo, s = orc.split(X, s=-10)
    assert s == -10
    rec = orc.reconstruct(hi, lo, s)
    assert np.max(np.abs(rec - X)) <= 2.0 ** -22 + 2.0 ** (-10 - 36)


# -------------------------------------------------------------- gemm -------

def _exact_dot(a_vals, b_vals):
    return sum((Fraction(x) * Fraction(y) for x, y in zip(a_vals, b_vals)), Fraction(0))


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8])
def test_split_gemm_brute_force_rationals(orc, n):
    """N <= 8: oracle C_split vs exact rational Eq. A_2 from independently-decoded planes."""
    for seed in range(6):
        for kind in ("uniform", "loguni"):
            A = numpy_matrix(kind, n, n + 1, seed=100 + seed)
            B = numpy_matrix(kind, n + 1, n, seed=200 + seed)
            A1, A2, sA = orc.split(A)
            B1, B2, sB = orc.split(B)
            # independent decode: numpy's float16 view
            a1, a2 = A1.view(np.float16).astype(np.float64), A2.view(np.float16).astype(np.float64)
            b1, b2 = B1.view(np.float16).astype(np.float64), B2.view(np.float16).astype(np.float64)
            for terms in (1, 3, 4):
                C = orc.split_gemm(A1, A2, sA, B1, B2, sB, terms)
                for i in range(n):
                    for j in range(n):
                        t11 = _exact_dot(a1[i], b1[:, j])
                        tm = _exact_dot(a1[i], b2[:, j]) + _exact_dot(a2[i], b1[:, j])
                        t22 = _exact_dot(a2[i], b2[:, j])
                        exact = t11
                        if terms >= 3:
                            exact += tm / 2 ** 11
                        if terms >= 4:
                            exact += t22 / 2 ** 22
                        exact *= Fraction(2) ** (sA + sB)
                        mag = (_exact_dot(np.abs(a1[i]) + np.abs(a2[i]), np.abs(b1[:, j]) + np.abs(b2[:, j]))
                               * Fraction(2) ** (sA + sB))
                        assert abs(Fraction(C[i, j]) - exact) <= mag * Fraction(n + 4, 2 ** 52)
            # FP64 reference GEMM vs exact rationals
            C64 = orc.gemm64(A, B)
            for i in range(n):
                for j in range(n):
                    ex = _exact_dot(A[i].astype(np.float64), B[:, j].astype(np.float64))
                    mag = _exact_dot(np.abs(A[i]).astype(np.float64), np.abs(B[:, j]).astype(np.float64))
                    assert abs(Fraction(C64[i, j]) - ex) <= mag * Fraction(n + 2, 2 ** 53)


def test_integer_inputs_exact(orc):
    """Entries in {-2..2}: A2 = B2 = 0 and C == exact integer product."""
    A = numpy_matrix("int2", 48, 200, seed=1)
    B = numpy_matrix("int2", 200, 40, seed=2)
    A1, A2, sA = orc.split(A)
    B1, B2, sB = orc.split(B)
    assert np.all(A2 & 0x7FFF == 0) and np.all(B2 & 0x7FFF == 0)
    exact = A.astype(np.int64) @ B.astype(np.int64)
    for terms in (1, 3, 4):
        assert np.array_equal(orc.split_gemm(A1, A2, sA, B1, B2, sB, terms), exact.astype(np.float64))
    assert np.array_equal(orc.gemm64(A, B), exact.astype(np.float64))


def test_gemm64_vs_numpy(orc):
    A = numpy_matrix("uniform", 33, 70, seed=3)
    B = numpy_matrix("uniform", 70, 21, seed=4)
    ref = A.astype(np.float64) @ B.astype(np.float64)
    assert np.max(np.abs(orc.gemm64(A, B) - ref)) <= 1e-13


def test_dropped_term_identity(orc):
    """4-term = 3-term + dropped term and its size bound."""
    A = numpy_matrix("uniform", 32, 32, seed=8)
    B = numpy_matrix("uniform", 32, 32, seed=9)
    A1, A2, sA = orc.split(A)
    B1, B2, sB = orc.split(B)
    c3 = orc.split_gemm(A1, A2, sA, B1, B2, sB, 3)
    c4 = orc.split_gemm(A1, A2, sA, B1, B2, sB, 4)
    d = orc.dropped_term(A2, sA, B2, sB)
    assert np.max(np.abs((c4 - c3) - d)) <= 1e-15 * np.max(np.abs(c3))
    # ||a2b2 A2B2|| = 2^-22 a1b1 ||A2 B2|| <= 2^-22 a1b1 ||A1||_F ||B1||_F  (|A2| <= |A1|)
    nA1 = np.linalg.norm(np.ldexp(orc.dec16(A1), sA))
    nB1 = np.linalg.norm(np.ldexp(orc.dec16(B1), sB))
    assert np.linalg.norm(d) <= 2.0 ** -22 * nA1 * nB1


def test_four_term_is_exact_when_the_split_is(orc):
    """Eq. A_1 with an exact residual (x = a1 A1 + a2 A2 exactly) makes the 4-term
    Eq. A_2 the exact product and the 3-term value the product minus exactly the dropped term
    (PAPER.md:21-24).  Entries +-16392 / +-16408 (s = 0): 16392 = 16384 + 8 ties to the even
    16384 (A2 = RN16(2^11 8) = 16384), 16408 = 16400 + 8 ties to 16416 (A2 = -16384) — hand-derived
    planes; the GPU's folded accumulator is pinned on the same inputs (test_gpu_fold.py)."""
    rng = np.random.default_rng(5)
    vals = np.array([16392, -16392, 16408, -16408], dtype=np.float32)
    A = vals[rng.integers(0, 4, (40, 2))]
    B = vals[rng.integers(0, 4, (2, 30))]
    a1, a2, sA = orc.split(A)
    assert sA == 0
    want1 = np.where(np.abs(A) == 16392, 16384.0, 16416.0) * np.sign(A)
    want2 = np.where(np.abs(A) == 16392, 16384.0, -16384.0) * np.sign(A)
    assert np.array_equal(orc.dec16(a1), want1) and np.array_equal(orc.dec16(a2), want2)
    exact = A.astype(np.float64) @ B.astype(np.float64)
    assert np.array_equal(orc.sgemm(A, B, terms=4), exact)
    b1, b2, sB = orc.split(B)
    drop = np.ldexp(orc.dec16(a2) @ orc.dec16(b2), sA + sB - 22)
    assert np.array_equal(orc.sgemm(A, B, terms=3), exact - drop)
    assert np.count_nonzero(drop) > 0


def test_accuracy_separation_n64(orc):
    """Config D1: 3-term error vs FP64 << naive FP16 (1-term) error, 20 seeds."""
    e3s, e1s, e4s = [], [], []
    for seed in range(20):
        A = numpy_matrix("uniform", 64, 64, seed=2 * seed)
        B = numpy_matrix("uniform", 64, 64, seed=2 * seed + 1)
        C64 = orc.gemm64(A, B)
        A1, A2, sA = orc.split(A)
        B1, B2, sB = orc.split(B)
        n = np.linalg.norm(C64)
        for terms, acc in ((1, e1s), (3, e3s), (4, e4s)):
            C = orc.split_gemm(A1, A2, sA, B1, B2, sB, terms)
            acc.append(np.linalg.norm(C - C64) / n)
    e1, e3, e4 = np.median(e1s), np.median(e3s), np.median(e4s)
    assert e3 < 2e-7 and e4 <= e3 * 1.05 and e1 > 1e-4
    assert all(a > 100 * b for a, b in zip(e1s, e3s))


def test_sampled_equals_full(orc):
    A = numpy_matrix("loguni", 40, 56, seed=21)
    B = numpy_matrix("loguni", 56, 36, seed=22)
    full = orc.sgemm(A, B, terms=3)
    rows = np.array([0, 7, 39, 12])
    cols = np.array([35, 0, 3])
    samp, sA, sB = orc.sgemm_sampled(A, B, rows, cols, terms=3)
    assert np.array_equal(samp, full[rows][:, cols])
    assert sA == orc.scale_exp(np.max(np.abs(A))) and sB == orc.scale_exp(np.max(np.abs(B)))


def test_nonfinite_rejected(orc):
    A = numpy_matrix("uniform", 4, 4, seed=0)
    A[2, 1] = np.nan
    with pytest.raises(ValueError, match="index 9"):
        orc.split(A)
