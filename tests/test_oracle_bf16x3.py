"""Pins of the oracle's bf16 x 3 split: the encoder against torch's
independent fp32 -> bfloat16 conversion, the split's reconstruction, and the 6-term product
against exact rationals."""
from fractions import Fraction

import numpy as np
import pytest
import torch

from workloads import numpy_matrix


def _torch_bf16_bits(x32):
    return torch.from_numpy(np.ascontiguousarray(x32, np.float32)).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)


def test_encbf16_vs_torch(orc):
    rng = np.random.Generator(np.random.PCG64(1))
    bits = rng.integers(0, 1 << 32, size=4_000_000, dtype=np.uint64).astype(np.uint32)
    # rounding boundaries: low 16 bits at/around the tie
    hi = rng.integers(0, 1 << 16, size=200_000, dtype=np.uint64).astype(np.uint32) << 16
    for low in (0x7FFF, 0x8000, 0x8001, 0xFFFF, 0):
        bits = np.concatenate([bits, hi | low])
    x = bits.view(np.float32)
    x = x[np.isfinite(x)]
    assert np.array_equal(orc.encbf16(x.astype(np.float64)), _torch_bf16_bits(x))


def test_decbf16_roundtrip(orc):
    h = np.arange(1 << 16, dtype=np.uint32).astype(np.uint16)
    d = orc.decbf16(h)
    fin = np.isfinite(d)
    assert np.array_equal(orc.encbf16(d[fin]), h[fin])


@pytest.mark.parametrize("kind,scale", [("uniform", 1.0), ("loguni", 1.0), ("uniform", 1e30), ("uniform", 1e-30)])
def test_split_bf16x3_reconstruction(orc, kind, scale):
    X = (numpy_matrix(kind, 64, 96, seed=4) * np.float32(scale)).astype(np.float32)
    p1, p2, p3 = orc.split_bf16x3(X)
    rec = orc.decbf16(p1) + orc.decbf16(p2) + orc.decbf16(p3)
    x = X.astype(np.float64)
    # each RN keeps >= 8 bits of the remaining residual: |x - rec| <= 2^-24 |x| (+ subnormal floor)
    assert np.all(np.abs(x - rec) <= 2.0 ** -24 * np.abs(x) + 2.0 ** -134)   # half the bf16 subnormal quantum
    # the leading plane alone is RN-bf16 of x (8 significant bits): rel error <= 2^-8
    assert np.all(np.abs(x - orc.decbf16(p1)) <= 2.0 ** -8 * np.abs(x))


def test_gemm_bf16x3_rationals(orc):
    for seed in range(4):
        A = numpy_matrix("uniform", 4, 6, seed=seed)
        B = numpy_matrix("loguni", 6, 3, seed=10 + seed)
        X, Y = orc.split_bf16x3(A), orc.split_bf16x3(B)
        C = orc.gemm_bf16x3_planes(X, Y)
        dx = [orc.decbf16(v) for v in X]
        dy = [orc.decbf16(v) for v in Y]
        for i in range(4):
            for j in range(3):
                ex = Fraction(0)
                mag = Fraction(0)
                for (p, q) in ((0, 0), (0, 1), (1, 0), (0, 2), (1, 1), (2, 0)):
                    for k in range(6):
                        t = Fraction(dx[p][i, k]) * Fraction(dy[q][k, j])
                        ex += t
                        mag += abs(t)
                assert abs(Fraction(C[i, j]) - ex) <= mag * Fraction(20, 2 ** 52)


def test_bf16x3_accuracy_near_fp32(orc):
    A = numpy_matrix("uniform", 64, 64, seed=1)
    B = numpy_matrix("uniform", 64, 64, seed=2)
    C64 = orc.gemm64(A, B)
    e = np.linalg.norm(orc.sgemm_bf16x3(A, B) - C64) / np.linalg.norm(C64)
    assert e < 1e-7
