"""Fused split of B inside the GEMM (Eq. A_1): the GEMM TMA-loads
B's fp32 tiles and converter warps write the B1/B2 planes into shared memory.  The converters use
the split kernels' arithmetic on the same values, and the MMAs run in the same K order, so C must
be BIT-identical to the separate-split path (mode 0) for every shape, layout and distribution;
the oracle pins it independently (E_or, E64)."""
import numpy as np
import pytest
import torch

import paper_2011_11188_b200 as s3
from workloads import torch_matrix

pytestmark = pytest.mark.gpu


def _h(mode):
    h = s3.Handle(0)
    h.set_fused_split(mode)
    return h


@pytest.fixture(scope="module")
def hf():
    return _h(2)     # fused whenever eligible


@pytest.fixture(scope="module")
def hs():
    return _h(0)     # separate split pass


def _bits(C):
    return C.view(torch.int32)


SHAPES = [(256, 512, 512), (300, 200, 500), (1000, 1030, 129), (257, 72, 4100), (64, 8, 64),
          (2048, 2048, 2048), (256, 8192, 1024), (100, 3000, 777), (1, 1, 1), (513, 1, 63), (7, 4096, 8192)]


@pytest.mark.parametrize("M,N,K", SHAPES)
@pytest.mark.parametrize("dist", ["uniform", "loguni"])
def test_fused_equals_separate(hf, hs, M, N, K, dist):
    A = torch_matrix("uniform", M, K, seed=21)
    B = torch_matrix(dist, K, N, seed=22)
    Cf = hf.sgemm(A, B).clone()
    Cs = hs.sgemm(A, B)
    assert torch.equal(_bits(Cf), _bits(Cs))


@pytest.mark.parametrize("transA,transB", [(0, 0), (1, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(300, 200, 500), (1000, 1030, 129), (256, 4096, 4096), (2048, 1024, 1024)])
def test_fused_all_transposes(hf, hs, transA, transB, M, N, K):
    A = torch_matrix("uniform", K if transA else M, M if transA else K, seed=23)
    B = torch_matrix("glorot", N if transB else K, K if transB else N, seed=24)
    Cf = hf.sgemm_ex(A, B, transA=bool(transA), transB=bool(transB)).clone()
    Cs = hs.sgemm_ex(A, B, transA=bool(transA), transB=bool(transB))
    assert torch.equal(_bits(Cf), _bits(Cs))


def test_fused_launch_count(hf, hs):
    """the fused call has no split kernel for B (one launch fewer)"""
    M, N, K = 256, 4096, 4096
    A = torch_matrix("uniform", M, K, seed=25)
    B = torch_matrix("uniform", K, N, seed=26)
    hf.sgemm(A, B)
    nf = hf.last_launch_count()
    hs.sgemm(A, B)
    ns = hs.last_launch_count()
    assert nf == ns - 1, (nf, ns)


def test_fused_strided_and_misaligned_b(hf, hs):
    """ld > N (column slice): fused; ld % 4 != 0 or a misaligned base: falls back (same bits)"""
    M, N, K = 384, 200, 640
    A = torch_matrix("uniform", M, K, seed=27)
    Bw = torch_matrix("uniform", K, N + 24, seed=28)
    for B in (Bw[:, :N], Bw[:, 1:N + 1], torch_matrix("uniform", K, N + 3, seed=29)[:, :N]):
        Cf = hf.sgemm(A, B).clone()
        Cs = hs.sgemm(A, B)
        assert torch.equal(_bits(Cf), _bits(Cs))


@pytest.mark.parametrize("scale", [0.0, 2.0 ** -100, 2.0 ** 100, 65504.0, 1e-38])
def test_fused_scale_edges(hf, hs, scale):
    """zero matrix (s = 0), tiny / huge magnitudes (s far from 0), fp32-subnormal inputs"""
    M, N, K = 256, 2048, 1024
    A = torch_matrix("uniform", M, K, seed=30)
    B = torch_matrix("uniform", K, N, seed=31) * scale
    Cf = hf.sgemm(A, B).clone()
    Cs = hs.sgemm(A, B)
    assert torch.equal(_bits(Cf), _bits(Cs))


def test_fused_vs_oracle(hf, orc):
    """independent pin: the oracle's 3-term emulation and the fp64 product"""
    M, N, K = 200, 1100, 900
    A = torch_matrix("uniform", M, K, seed=32)
    B = torch_matrix("loguni", K, N, seed=33)
    C = hf.sgemm(A, B).cpu().numpy()
    An, Bn = A.cpu().numpy(), B.cpu().numpy()
    Cs = orc.sgemm(An, Bn, terms=3)
    e_or = np.linalg.norm(C - Cs) / np.linalg.norm(Cs)
    C64 = orc.gemm64(An, Bn)
    e64 = np.linalg.norm(C - C64) / (np.linalg.norm(An.astype(np.float64)) * np.linalg.norm(Bn.astype(np.float64)))
    assert e_or <= 1e-6 and e64 <= 2e-6, (e_or, e64)


def test_fused_split_k_writes_scale(hf, hs):
    """split-K shapes: the tail reduction reads the B scale exponent the fused GEMM stored"""
    M, N, K = 256, 1024, 8192       # 4 tiles < 74 pairs: every tile cut into K slices
    A = torch_matrix("uniform", M, K, seed=34) * 3.0
    B = torch_matrix("uniform", K, N, seed=35) * 1000.0
    Cf = hf.sgemm(A, B).clone()
    Cs = hs.sgemm(A, B)
    assert torch.equal(_bits(Cf), _bits(Cs))


def test_fused_graph_replay(hf, hs):
    """captured fused call replays bitwise, also after the inputs (and so the scales) change"""
    M, N, K = 256, 4096, 2048
    A = torch_matrix("uniform", M, K, seed=36)
    B = torch_matrix("uniform", K, N, seed=37)
    C = torch.empty(M, N, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        hf.sgemm(A, B, out=C)      # warm-up (workspace) outside the capture
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            hf.sgemm(A, B, out=C)
    torch.cuda.current_stream().wait_stream(s)
    for seed, scale in ((38, 1.0), (39, 2.0 ** 20)):
        A.copy_(torch_matrix("uniform", M, K, seed=seed))
        B.copy_(torch_matrix("loguni", K, N, seed=seed + 100) * scale)
        g.replay()
        torch.cuda.synchronize()
        Cs = hs.sgemm(A, B)
        assert torch.equal(_bits(C), _bits(Cs))


def test_fused_mode_validation(hf):
    with pytest.raises(s3.Split3Error):
        hf.set_fused_split(3)
    with pytest.raises(s3.Split3Error):
        hf.set_fused_split(1, -1)


def test_fused_nonfinite_b(hf, hs):
    """Inf / NaN in B: skipped by the max, propagated by the converters exactly as by the split
    kernel (bitwise, NaN payloads included); SPLIT3_CHECK_FINITE reports the first bad index"""
    M, N, K = 256, 2048, 1024
    A = torch_matrix("uniform", M, K, seed=52)
    B = torch_matrix("uniform", K, N, seed=53)
    B[10, 7] = float("inf")
    B[500, 1000] = float("nan")
    Cf = hf.sgemm(A, B).clone()
    Cs = hs.sgemm(A, B)
    assert torch.equal(_bits(Cf), _bits(Cs))
    assert not torch.isfinite(Cf[:, 7]).any() and torch.isnan(Cf[:, 1000]).all()
    with pytest.raises(s3.NotFiniteError) as ei:
        hf.sgemm(A, B, check_finite=True)
    assert ei.value.index == M * K + 10 * N + 7


@pytest.mark.parametrize("M,N,K", [(256, 512, 512), (1000, 1030, 129), (257, 72, 4100), (7, 4096, 8192),
                                   (2048, 2048, 2048), (1, 1, 1)])
@pytest.mark.parametrize("dist", ["uniform", "loguni"])
def test_fused_kmajor_equals_separate(hf, hs, M, N, K, dist):
    """B given as B^T (stored N x K): the K-major in-place layout (8-row groups, SBO 2 KB)"""
    A = torch_matrix("uniform", M, K, seed=54)
    Bt = torch_matrix(dist, N, K, seed=55)
    Cf = hf.sgemm_ex(A, Bt, transB=True).clone()
    nf = hf.last_launch_count()
    Cs = hs.sgemm_ex(A, Bt, transB=True)
    assert torch.equal(_bits(Cf), _bits(Cs))
    if M * K + N * K > 4 << 20:
        assert nf == hs.last_launch_count() - 1      # no transposing split of B
