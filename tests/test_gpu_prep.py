"""One-launch front end for small problems (max-abs of both operands, grid-wide barrier, both
splits in one cooperative kernel) against the separate max-abs / split kernels
(SPLIT3_PREP_MAX=0).  Same scales and planes -> C must be BIT-identical."""
import os

import pytest
import torch

import paper_2011_11188_b200 as s3
from workloads import torch_matrix

pytestmark = pytest.mark.gpu


def _handle(prep_max: int | None):
    old = os.environ.get("SPLIT3_PREP_MAX")
    if prep_max is None:
        os.environ.pop("SPLIT3_PREP_MAX", None)
    else:
        os.environ["SPLIT3_PREP_MAX"] = str(prep_max)
    try:
        h = s3.Handle(0)
        h.set_fused_split(0)     # this file compares the front ends of the separate-split path
        return h
    finally:
        if old is None:
            os.environ.pop("SPLIT3_PREP_MAX", None)
        else:
            os.environ["SPLIT3_PREP_MAX"] = old


@pytest.fixture(scope="module")
def hp():
    return _handle(1 << 40)      # one-launch front end at every size


@pytest.fixture(scope="module")
def hs():
    return _handle(0)            # separate kernels


@pytest.mark.parametrize("transA,transB", [(0, 0), (1, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (64, 64, 64), (300, 200, 500), (1000, 1030, 129),
                                   (257, 72, 4100), (3, 5000, 7), (2048, 2048, 2048)])
@pytest.mark.parametrize("kw", [{}, {"four_term": True}, {"one_term": True}])
def test_prep_equals_separate_kernels(hp, hs, transA, transB, M, N, K, kw):
    A = torch_matrix("loguni", K if transA else M, M if transA else K, seed=21)
    B = torch_matrix("uniform", N if transB else K, K if transB else N, seed=22)
    Cp = hp.sgemm_ex(A, B, transA=bool(transA), transB=bool(transB), **kw).clone()
    Cs = hs.sgemm_ex(A, B, transA=bool(transA), transB=bool(transB), **kw)
    assert torch.equal(Cp.view(torch.int32), Cs.view(torch.int32))


def test_prep_strided_and_misaligned(hp, hs):
    """ld > cols and a base pointer 4 bytes off 16-B alignment (scalar paths of the kernel)."""
    M, N, K = 130, 98, 77
    Aw = torch_matrix("uniform", M, K + 5, seed=23)
    Bw = torch_matrix("uniform", K, N + 3, seed=24)
    A, B = Aw[:, 1:K + 1], Bw[:, :N]
    Cp = hp.sgemm_ex(A, B).clone()
    Cs = hs.sgemm_ex(A, B)
    assert torch.equal(Cp.view(torch.int32), Cs.view(torch.int32))


def test_prep_graph_replays_track_new_inputs(hp, hs):
    """Under capture the library takes the separate front-end kernels (faster replays); the graph,
    replayed with inputs whose scales change, matches fresh eager calls (which take the one-launch
    front end) bitwise."""
    M, N, K = 512, 384, 640
    A = torch_matrix("uniform", M, K, seed=25)
    B = torch_matrix("uniform", K, N, seed=26)
    C = torch.empty((M, N), device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        hp.sgemm(A, B, out=C)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            hp.sgemm(A, B, out=C)
    torch.cuda.synchronize()
    for step, (sa, sb) in enumerate([(1.0, 1.0), (1e4, 1.0), (1.0, 3e-7), (0.5, 2.0), (1.0, 1.0)]):
        A.copy_(torch_matrix("uniform", M, K, seed=30 + step) * sa)
        B.copy_(torch_matrix("uniform", K, N, seed=40 + step) * sb)
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(C.view(torch.int32), hs.sgemm(A, B).view(torch.int32)), step


def test_prep_launch_count(hp, hs):
    A = torch_matrix("uniform", 256, 256, seed=27)
    B = torch_matrix("uniform", 256, 256, seed=28)
    hp.sgemm(A, B)
    hs.sgemm(A, B)
    assert hs.last_launch_count() - hp.last_launch_count() == 2   # 3 front-end kernels -> 1
