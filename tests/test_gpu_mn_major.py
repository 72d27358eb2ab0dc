"""MN-major operand planes (default: a row-major fp32 B and a transposed fp32 A are split without
a transpose, and the GEMM reads K x N / K x M planes with MN-major smem descriptors) against the
K-major path (SPLIT3_MN_MAJOR=0: transposing splits into N x K / M x K planes).  Same plane values,
same MMA K order -> C must be BIT-identical."""
import os

import numpy as np
import pytest
import torch

import paper_2011_11188_b200 as s3
from workloads import torch_matrix

pytestmark = pytest.mark.gpu


def _handle(b_mn: bool):
    old = os.environ.get("SPLIT3_MN_MAJOR")
    os.environ["SPLIT3_MN_MAJOR"] = "1" if b_mn else "0"
    try:
        return s3.Handle(0)
    finally:
        if old is None:
            os.environ.pop("SPLIT3_MN_MAJOR", None)
        else:
            os.environ["SPLIT3_MN_MAJOR"] = old


@pytest.fixture(scope="module")
def hm():
    return _handle(True)


@pytest.fixture(scope="module")
def hk():
    return _handle(False)


@pytest.mark.parametrize("M,N,K", [(512, 512, 512), (300, 200, 500), (1000, 1030, 129), (257, 72, 4100),
                                   (64, 8, 64), (2048, 2048, 2048), (256, 8192, 1024)])
@pytest.mark.parametrize("kw", [{}, {"four_term": True}, {"one_term": True}, {"bf16x3": True}])
def test_b_mn_equals_k_major(hm, hk, M, N, K, kw):
    A = torch_matrix("uniform", M, K, seed=3)
    B = torch_matrix("loguni", K, N, seed=4)
    Cm = hm.sgemm(A, B, **kw).clone()
    Ck = hk.sgemm(A, B, **kw)
    assert torch.equal(Cm.view(torch.int32), Ck.view(torch.int32))


@pytest.mark.parametrize("transA,transB", [(0, 0), (1, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("kw", [{}, {"four_term": True}, {"one_term": True}, {"bf16x3": True}])
@pytest.mark.parametrize("M,N,K", [(300, 200, 500), (1000, 1030, 129), (2048, 1024, 1024)])
def test_mn_major_all_transposes(hm, hk, transA, transB, kw, M, N, K):
    A = torch_matrix("uniform", K if transA else M, M if transA else K, seed=13)
    B = torch_matrix("glorot", N if transB else K, K if transB else N, seed=14)
    Cm = hm.sgemm_ex(A, B, transA=bool(transA), transB=bool(transB), **kw).clone()
    Ck = hk.sgemm_ex(A, B, transA=bool(transA), transB=bool(transB), **kw)
    assert torch.equal(Cm.view(torch.int32), Ck.view(torch.int32))


def test_b_mn_with_transposed_a_and_strided_b(hm, hk):
    """op(A) = A^T and a B with ld > N (a column slice of a wider matrix)."""
    M, N, K = 384, 200, 640
    At = torch_matrix("uniform", K, M, seed=5)
    Bw = torch_matrix("uniform", K, N + 24, seed=6)
    B = Bw[:, :N]
    Cm = hm.sgemm_ex(At, B, transA=True).clone()
    Ck = hk.sgemm_ex(At, B, transA=True)
    assert torch.equal(Cm.view(torch.int32), Ck.view(torch.int32))


def test_b_mn_host_path(hm, hk):
    """split3_sgemm_host (row-block pipeline) with both B layouts, and against the device path."""
    M, N, K = 1700, 900, 1100
    A = torch_matrix("uniform", M, K, seed=7)
    B = torch_matrix("uniform", K, N, seed=8)
    Cm = hm.sgemm_host(A.cpu().numpy(), B.cpu().numpy())
    Ck = hk.sgemm_host(A.cpu().numpy(), B.cpu().numpy())
    assert np.array_equal(Cm.view(np.int32), Ck.view(np.int32))
    # the device path may cut this shape into split-K slices (the host pipeline does not): same
    # planes, different summation order -> compare to a tolerance, not bitwise
    Cd = hm.sgemm(A, B).cpu().numpy().astype(np.float64)
    assert np.linalg.norm(Cm - Cd) / np.linalg.norm(Cd) < 1e-6
