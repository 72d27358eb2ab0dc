"""Seeded synthetic input generators shared by tests/, bench.py and smoke().

Holds none of the method's arithmetic: it only draws FP32 matrices with the
shapes and value distributions of BASELINE.json's configs (recipes in
DESIGN.md §4).  Both the oracle side and the CUDA side receive the SAME arrays
from here; neither generates its own inputs.

Kinds:
  uniform   A = 2*U[0,1) - 1                                  (configs D1, D2, D5)
  glorot    W ~ U[-sqrt(6/(fan_in+fan_out)), +...]            (config D3 weights)
  loguni    x = +-2^u, u ~ U(-20, 20), sign +-1 w.p. 1/2       (config D4)
  int2      x in {-2,-1,0,1,2} uniformly                       (exactness pin)
  fp16      fp16-representable values of magnitude < 2^15     (A2 == 0 pin)
"""
from __future__ import annotations

import numpy as np

KINDS = ("uniform", "glorot", "loguni", "int2", "fp16")


def numpy_matrix(kind: str, rows: int, cols: int, seed: int) -> np.ndarray:
    """Row-major float32 matrix of the given kind, from numpy's PCG64(seed)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    if kind == "uniform":
        return (2.0 * rng.random((rows, cols), dtype=np.float32) - 1.0).astype(np.float32)
    if kind == "glorot":
        lim = np.sqrt(6.0 / (rows + cols))
        return ((2.0 * rng.random((rows, cols)) - 1.0) * lim).astype(np.float32)
    if kind == "loguni":
        u = rng.uniform(-20.0, 20.0, size=(rows, cols))
        sgn = np.where(rng.random((rows, cols)) < 0.5, -1.0, 1.0)
        return (sgn * np.exp2(u)).astype(np.float32)
    if kind == "int2":
        return rng.integers(-2, 3, size=(rows, cols)).astype(np.float32)
    if kind == "fp16":
        # uniform over binary16 bit patterns with exponent field < 30 (|x| < 2^15)
        bits = rng.integers(0, 1 << 16, size=(rows, cols), dtype=np.uint32).astype(np.uint16)
        exp = (bits >> 10) & 0x1F
        bits = np.where(exp >= 30, bits & ~np.uint16(0x1000), bits).astype(np.uint16)
        return bits.view(np.float16).astype(np.float32)
    raise ValueError(f"unknown kind {kind!r}")


def torch_matrix(kind: str, rows: int, cols: int, seed: int, device="cuda"):
    """Same distributions drawn with torch's generator on `device` (large sizes).

    The stream differs from numpy_matrix for the same seed; a test always hands
    the SAME tensor (copied to host where needed) to both sides.
    """
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    if kind == "uniform":
        t = torch.rand((rows, cols), generator=g, device=device, dtype=torch.float32)
        return t.mul_(2.0).sub_(1.0)
    if kind == "glorot":
        lim = float(np.sqrt(6.0 / (rows + cols)))
        t = torch.rand((rows, cols), generator=g, device=device, dtype=torch.float32)
        return t.mul_(2.0 * lim).sub_(lim)
    if kind == "loguni":
        u = torch.rand((rows, cols), generator=g, device=device, dtype=torch.float32)
        u = u.mul_(40.0).sub_(20.0)
        sgn = torch.rand((rows, cols), generator=g, device=device) < 0.5
        t = torch.exp2(u)
        return torch.where(sgn, -t, t)
    if kind == "int2":
        return torch.randint(-2, 3, (rows, cols), generator=g, device=device).to(torch.float32)
    if kind == "fp16":
        bits = torch.randint(0, 1 << 16, (rows, cols), generator=g, device=device, dtype=torch.int32)
        exp = (bits >> 10) & 0x1F
        bits = torch.where(exp >= 30, bits & ~0x1000, bits)
        return bits.to(torch.int16).view(torch.float16).to(torch.float32)
    raise ValueError(f"unknown kind {kind!r}")


def make_blobs(n: int, classes: int, dim: int, separation: float, seed: int):
    """Seeded Gaussian clusters (SPEC.md mlp make_blobs): class means at distance ~separation,
    unit-variance noise.  Returns (X float32 n x dim, y int32 n)."""
    if classes < 2:
        raise ValueError("classes must be >= 2")
    rng = np.random.Generator(np.random.PCG64(seed))
    centers = rng.standard_normal((classes, dim))
    centers *= (separation / np.sqrt(2.0)) / np.linalg.norm(centers, axis=1, keepdims=True)
    y = rng.integers(0, classes, size=n).astype(np.int32)
    X = (centers[y] + rng.standard_normal((n, dim))).astype(np.float32)
    return X, y
