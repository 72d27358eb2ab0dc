"""Host-buffer pipeline (split3_sgemm_host): A arrives in row blocks, each split with
its own scale exponent; a block whose exponent is below the per-matrix one (reading R1) gives the
per-matrix bits by exact power-of-two scaling unless it holds a nonzero |a| < 2^(sA-12), in which
case the library redoes it.  C must be BIT-identical to the one-block host call (per-matrix scale,
same whole-tile GEMM plan) in every case, and match the device-buffer call (whose small problems
may use split-K slices, another summation order) to the oracle tolerance."""
import os

import numpy as np
import pytest
import torch

import paper_2011_11188_b200 as s3
from workloads import numpy_matrix

pytestmark = pytest.mark.gpu


def _handle(blocks):
    old = os.environ.get("SPLIT3_HOST_BLOCKS")
    os.environ["SPLIT3_HOST_BLOCKS"] = str(blocks)
    try:
        return s3.Handle(0)
    finally:
        if old is None:
            os.environ.pop("SPLIT3_HOST_BLOCKS", None)
        else:
            os.environ["SPLIT3_HOST_BLOCKS"] = old


@pytest.fixture(scope="module")
def hb():
    return _handle(4)


@pytest.fixture(scope="module")
def hd():
    return _handle(1)     # one block: the per-matrix scale for all of A


def _device(hd, A, B, **kw):
    C1 = hd.sgemm_host(A, B, **kw)
    Cd = hd.sgemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), **kw).cpu().numpy()
    fin = np.isfinite(Cd)
    assert np.array_equal(fin, np.isfinite(C1))
    if fin.any():
        d = Cd[fin].astype(np.float64)
        assert np.linalg.norm(C1[fin] - d) <= 1e-6 * max(np.linalg.norm(d), 1e-300)
    return C1


def _same(x, y):
    return np.array_equal(x.view(np.int32), y.view(np.int32))


@pytest.mark.parametrize("kw", [{}, {"four_term": True}, {"one_term": True}])
@pytest.mark.parametrize("M,N,K", [(2048, 512, 700), (1100, 300, 257), (1024, 1024, 64)])
def test_blocks_equal_device(hb, hd, M, N, K, kw):
    A = numpy_matrix("uniform", M, K, seed=40)
    B = numpy_matrix("glorot", K, N, seed=41)
    assert _same(hb.sgemm_host(A, B, **kw), _device(hd, A, B, **kw))


def test_block_exponents_differ_no_redo(hb, hd):
    """block 0 five binades below the rest: its planes are the per-matrix ones x 2^5 exactly"""
    M, N, K = 2048, 512, 700
    A = numpy_matrix("uniform", M, K, seed=42)
    A[:512] = np.sign(A[:512]) * np.maximum(np.abs(A[:512]), np.float32(2.0 ** -20))
    A[:512] *= 2.0 ** -5
    assert np.abs(A).min() >= 2.0 ** -27 and np.abs(A).max() >= 0.5   # nothing below 2^(sA-12), sA = -15
    B = numpy_matrix("loguni", K, N, seed=43)
    r0 = hb.host_redo_count()
    C = hb.sgemm_host(A, B)
    assert hb.host_redo_count() == r0
    assert _same(C, _device(hd, A, B))


@pytest.mark.parametrize("tiny", [2.0 ** -40, 2.0 ** -30, 1e-45])
def test_block_with_tiny_entry_is_redone(hb, hd, tiny):
    """a low-exponent block with a nonzero entry below 2^(sA-12) is redone with the per-matrix scale"""
    M, N, K = 2048, 512, 700
    A = numpy_matrix("uniform", M, K, seed=44)
    A[:512] *= 2.0 ** -5
    A[3, 5] = np.float32(tiny)
    A[100, 7] = -np.float32(tiny) * 3
    B = numpy_matrix("uniform", K, N, seed=45)
    r0 = hb.host_redo_count()
    C = hb.sgemm_host(A, B)
    assert hb.host_redo_count() == r0 + 1
    assert _same(C, _device(hd, A, B))


def test_wide_range_blocks(hb, hd):
    """log-uniform magnitudes (2^-20..2^20) in every block: exponents and tiny entries everywhere"""
    M, N, K = 2048, 384, 512
    A = numpy_matrix("loguni", M, K, seed=46)
    A[512:1024] *= 2.0 ** -30
    B = numpy_matrix("loguni", K, N, seed=47)
    assert _same(hb.sgemm_host(A, B), _device(hd, A, B))


def test_zero_and_nonfinite_blocks(hb, hd):
    """an all-zero block (exponent 0) and a block with Inf/NaN (skipped by the max, propagated)"""
    M, N, K = 2048, 256, 320
    A = numpy_matrix("uniform", M, K, seed=48)
    A[:512] = 0.0
    A[1500, 3] = np.inf
    A[1700, 9] = np.nan
    B = numpy_matrix("uniform", K, N, seed=49)
    C = hb.sgemm_host(A, B)
    Cd = _device(hd, A, B)
    assert _same(C, Cd)
    assert np.isnan(C[1700]).all() and not np.isfinite(C[1500]).any()


def test_auto_blocks_with_tail(hd):
    """automatic blocking (4 blocks, the last cut into 1/2 + 1/4 + 1/4) with differing block scales"""
    M, N, K = 8192, 16384, 320
    A = numpy_matrix("uniform", M, K, seed=50)
    A[2048:4096] *= 2.0 ** -3
    A[7000, 1] = np.float32(2.0 ** -45)       # a tiny entry in a tail block with the top exponent
    B = numpy_matrix("uniform", K, N, seed=51)
    h = s3.Handle(0)
    C = h.sgemm_host(A, B)
    assert h.last_launch_count() > 6 * 3          # 6 row blocks: max/min, split, GEMM each
    assert _same(C, hd.sgemm_host(A, B))


@pytest.mark.parametrize("case", ["plain", "b_panel_scaled", "b_tiny", "a_and_b_tiny"])
def test_2d_schedule_b_panels(hd, case):
    """automatic 2-D schedule (2 B column panels interleaved with the first A blocks, each panel
    split with its own exponent): bitwise equal to the one-block call, pieces redone when needed"""
    M, N, K = 8192, 16384, 256
    A = numpy_matrix("uniform", M, K, seed=56)
    B = numpy_matrix("uniform", K, N, seed=57)
    half = N // 2                                    # B panel 0
    if case != "plain":                              # panel 0 six binades below panel 1
        B[:, :half] = np.sign(B[:, :half]) * np.maximum(np.abs(B[:, :half]), np.float32(2.0 ** -20))
        B[:, :half] *= 2.0 ** -6
    if case in ("b_tiny", "a_and_b_tiny"):
        B[17, 100] = np.float32(2.0 ** -50)         # a tiny entry in the low-exponent panel
    if case == "a_and_b_tiny":
        A[:2048] = np.sign(A[:2048]) * np.maximum(np.abs(A[:2048]), np.float32(2.0 ** -20))
        A[:2048] *= 2.0 ** -4
        A[5, 5] = np.float32(2.0 ** -60)
    h = s3.Handle(0)
    r0 = h.host_redo_count()
    C = h.sgemm_host(A, B)
    redo = h.host_redo_count() - r0
    assert redo == {"plain": 0, "b_panel_scaled": 0, "b_tiny": 1, "a_and_b_tiny": 2}[case], redo
    assert _same(C, hd.sgemm_host(A, B))
