"""Fused split of A inside the GEMM (SURVEY §8f NEXT #2 for the second operand; Eq. A_1,
PAPER.md:4-8): the call computes the transposed problem C^T = B^T A^T, whose fused operand is
A^T — A's fp32 tiles are TMA-loaded and split in shared memory by the converter warps, B's planes
are the tensor core's A operand — and the epilogue (and the split-K tail reduction) writes every
C^T tile transposed into C.

Pins: (1) the oracle — E_or, E64 and the per-element bound on every element; (2) bitwise equality
with the same transposed problem computed from separately split planes (split3_sgemm_ex with
transA = transB = 1, fusion off), which fixes the planes, the K order and the epilogue.  Not
bitwise: the ordinary (untransposed) call.  Every element is the same sum of the same exact
products in the same k-block order, but the tensor core accumulates a K = 16 step differently when
the two operands swap roles (measured: the bits differ; DESIGN.md §3 R9), so the two are compared
with the oracle tolerance and the per-element bound instead."""
import numpy as np
import pytest
import torch

import paper_2011_11188_b200 as s3
from split3_bounds import _assert_elementwise
from workloads import torch_matrix

pytestmark = pytest.mark.gpu


def _h(mode_a, mode_b):
    h = s3.Handle(0)
    h.set_fused_split_a(mode_a)
    h.set_fused_split(mode_b)
    return h


@pytest.fixture(scope="module")
def ha():
    return _h(2, 0)     # fused A whenever eligible


@pytest.fixture(scope="module")
def hs():
    return _h(0, 0)     # separate split passes


def _bits(C):
    return C.view(torch.int32)


def _ref_t(hs, A, B):
    """(B^T A^T)^T from separately split planes: the bits the fused-A path must reproduce"""
    return hs.sgemm_ex(B, A, transA=True, transB=True).t().contiguous()


# K % 4 == 0 (A's rows 16-B aligned) for the fused path; (4100, 72, 257), (1, 1, 1), (1, 513, 63) and
# (4096, 7, 8192) (ld % 4 != 0 or ldc % 4 != 0) take the fallback
SHAPES = [(512, 256, 512), (300, 200, 500), (1030, 1000, 132), (4100, 72, 260), (4100, 72, 257), (64, 8, 64),
          (2048, 2048, 2048), (8192, 256, 1024), (3000, 100, 780), (1, 1, 1), (1, 513, 63), (4096, 7, 8192),
          (4096, 1024, 1024), (4096, 8, 8192)]


def _eligible(lda, ldc):
    """fused A needs A's rows and C's rows 16-B aligned (contiguous tensors: ld % 4 == 0)"""
    return lda % 4 == 0 and ldc % 4 == 0


@pytest.mark.parametrize("M,N,K", SHAPES)
@pytest.mark.parametrize("dist", ["uniform", "loguni"])
def test_fused_a_equals_transposed_and_plain(ha, hs, M, N, K, dist):
    A = torch_matrix(dist, M, K, seed=61)
    B = torch_matrix("uniform", K, N, seed=62)
    Ca = ha.sgemm(A, B).clone()
    assert bool(ha.last_path() & 2) == _eligible(K, N)      # SPLIT3_PATH_FUSED_A
    Ct = _ref_t(hs, A, B)          # (B^T A^T)^T, separate split
    Cs = hs.sgemm(A, B)            # untransposed: same sums, another in-MMA order (module docstring)
    assert torch.equal(_bits(Ca), _bits(Ct if _eligible(K, N) else Cs))
    Cs64, Ca64 = Cs.double(), Ca.double()
    assert float((Ca64 - Cs64).norm() / Cs64.norm().clamp_min(1e-300)) <= 1e-6


@pytest.mark.parametrize("M,N,K", [(300, 200, 500), (1030, 1000, 132), (4100, 72, 260), (2304, 256, 4096)])
def test_fused_a_vs_oracle(ha, orc, M, N, K):
    A = torch_matrix("loguni", M, K, seed=63)
    B = torch_matrix("uniform", K, N, seed=64)
    C = ha.sgemm(A, B).cpu().numpy()
    An, Bn = A.cpu().numpy(), B.cpu().numpy()
    Cs = orc.sgemm(An, Bn, terms=3)
    C64 = orc.gemm64(An, Bn)
    e_or = np.linalg.norm(C - Cs) / np.linalg.norm(Cs)
    e64 = np.linalg.norm(C - C64) / (np.linalg.norm(An.astype(np.float64)) * np.linalg.norm(Bn.astype(np.float64)))
    assert e_or <= 1e-6 and e64 <= 2e-6, (e_or, e64)
    _assert_elementwise(orc, C, Cs, An, Bn, 3)


@pytest.mark.parametrize("transA,transB", [(0, 0), (1, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(300, 200, 500), (1030, 1000, 132), (4096, 256, 4096), (2048, 1024, 1024)])
def test_fused_a_all_transposes(ha, hs, transA, transB, M, N, K):
    A = torch_matrix("uniform", K if transA else M, M if transA else K, seed=65)
    B = torch_matrix("glorot", N if transB else K, K if transB else N, seed=66)
    Ca = ha.sgemm_ex(A, B, transA=bool(transA), transB=bool(transB)).clone()
    if _eligible(A.stride(0), N):
        # the transposed problem with separately split planes: op(B)^T op(A)^T
        ref = hs.sgemm_ex(B, A, transA=not transB, transB=not transA).t().contiguous()
    else:
        ref = hs.sgemm_ex(A, B, transA=bool(transA), transB=bool(transB))
    assert torch.equal(_bits(Ca), _bits(ref))


def test_fused_a_presplit_b(ha, hs):
    """B pre-split (K-major planes of role 1, or the stored matrix's planes): still fused A"""
    M, N, K = 2048, 512, 1536
    A = torch_matrix("uniform", M, K, seed=67)
    B = torch_matrix("glorot", K, N, seed=68)
    ref = _ref_t(hs, A, B)
    for W in (ha.presplit(B, role=1), ha.presplit_stored(B)):
        Ca = ha.sgemm_ex(A, W)
        na = ha.last_launch_count()
        assert torch.equal(_bits(Ca), _bits(ref))
        assert na <= 3, na          # max-abs of A + GEMM (+ split-K reduction): no split kernel at all


def test_fused_a_launch_count(ha, hs):
    """the fused call has no split kernel for A (one launch fewer)"""
    M, N, K = 4096, 256, 4096
    A = torch_matrix("uniform", M, K, seed=69)
    B = torch_matrix("uniform", K, N, seed=70)
    ha.sgemm(A, B)
    na = ha.last_launch_count()
    hs.sgemm(A, B)
    assert na == hs.last_launch_count() - 1, (na, hs.last_launch_count())


def test_fused_a_auto_selection():
    """mode 1: fused A when N <= 2048 and N < M (A is the larger operand), fused B when M <= 2048
    and M <= N (the default handle: fused B only, never fused A)"""
    h = _h(1, 1)
    hd = s3.Handle(0)
    hs = _h(0, 0)
    for (M, N, K), fewer in (((4096, 1024, 1024), True), ((1024, 4096, 1024), True), ((8192, 4096, 512), False)):
        A = torch_matrix("uniform", M, K, seed=71)
        B = torch_matrix("uniform", K, N, seed=72)
        C = h.sgemm(A, B).clone()
        n = h.last_launch_count()
        Cs = hs.sgemm(A, B)
        ns = hs.last_launch_count()
        # fused A reproduces the transposed problem's bits, fused B the untransposed call's
        ref = _ref_t(hs, A, B) if N < M and N <= 2048 else Cs
        assert torch.equal(_bits(C), _bits(ref))
        assert (n == ns - 1) == fewer, (M, N, K, n, ns)
        assert torch.equal(_bits(hd.sgemm(A, B)), _bits(Cs))     # default: the untransposed bits


def test_fused_a_strided_and_misaligned(ha, hs):
    """A with ld > K: fused; A with ld % 4 != 0, or C not TMA-storable (ldc % 4 != 0): falls back
    to the separate split (same bits either way)"""
    M, N, K = 1200, 200, 640
    Aw = torch_matrix("uniform", M, K + 12, seed=73)
    B = torch_matrix("uniform", K, N, seed=74)
    for A, fused in ((Aw[:, :K], True), (Aw[:, 3:K + 3], False), (torch_matrix("uniform", M, K + 3, seed=75)[:, :K], False)):
        Ca = ha.sgemm(A, B).clone()
        ref = _ref_t(hs, A, B) if fused else hs.sgemm(A, B)
        assert torch.equal(_bits(Ca), _bits(ref))
    A = Aw[:, :K]
    Cbig = torch.full((M, N + 3), 7.0, device="cuda")      # ldc % 4 != 0: no TMA store, no fused A
    ha.sgemm(A, B, out=Cbig[:, 1:1 + N])
    assert torch.equal(_bits(Cbig[:, 1:1 + N].contiguous()), _bits(hs.sgemm(A, B)))
    assert torch.all(Cbig[:, 0] == 7.0) and torch.all(Cbig[:, N + 1:] == 7.0)
    Cbig = torch.full((M, N + 4), 7.0, device="cuda")       # ldc % 4 == 0, 16-B aligned column offset: fused
    ha.sgemm(A, B, out=Cbig[:, 4:4 + N])
    assert torch.equal(_bits(Cbig[:, 4:4 + N].contiguous()), _bits(_ref_t(hs, A, B)))
    assert torch.all(Cbig[:, :4] == 7.0)


def test_fused_a_split_k_tail(ha, hs):
    """few tiles: every tile of C^T cut into K slices, reduced and written transposed"""
    for M, N, K in ((1024, 256, 8192), (300, 20, 16384), (2304, 256, 4096)):
        A = torch_matrix("uniform", M, K, seed=76) * 3.0
        B = torch_matrix("uniform", K, N, seed=77) * 1000.0
        Ca = ha.sgemm(A, B).clone()
        assert torch.equal(_bits(Ca), _bits(_ref_t(hs, A, B))), (M, N, K)


def test_fused_a_nonfinite(ha, hs):
    M, N, K = 2048, 256, 1024
    A = torch_matrix("uniform", M, K, seed=78)
    B = torch_matrix("uniform", K, N, seed=79)
    A[10, 7] = float("inf")
    A[500, 1000] = float("nan")
    Ca = ha.sgemm(A, B).clone()
    assert torch.equal(_bits(Ca), _bits(_ref_t(hs, A, B)))
    assert not torch.isfinite(Ca[10]).any() and torch.isnan(Ca[500]).all()
    with pytest.raises(s3.NotFiniteError) as ei:
        ha.sgemm(A, B, check_finite=True)
    assert ei.value.index == 10 * K + 7


def test_fused_a_graph_replay(ha, hs):
    M, N, K = 4096, 256, 2048
    A = torch_matrix("uniform", M, K, seed=80)
    B = torch_matrix("uniform", K, N, seed=81)
    C = torch.empty(M, N, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        ha.sgemm(A, B, out=C)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            ha.sgemm(A, B, out=C)
    torch.cuda.current_stream().wait_stream(s)
    for seed, scale in ((82, 1.0), (83, 2.0 ** -30)):
        A.copy_(torch_matrix("loguni", M, K, seed=seed) * scale)
        B.copy_(torch_matrix("uniform", K, N, seed=seed + 100))
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(_bits(C), _bits(_ref_t(hs, A, B)))


def test_fused_a_mode_validation(ha):
    with pytest.raises(s3.Split3Error):
        ha.set_fused_split_a(3)
    with pytest.raises(s3.Split3Error):
        ha.set_fused_split_a(1, -1)
