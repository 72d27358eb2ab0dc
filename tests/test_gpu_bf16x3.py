"""NEXT #4: the bf16 x 3 variant (SPLIT3_BF16X3) vs the oracle's bf16x3 emulation and FP64."""
import numpy as np
import pytest
import torch

from workloads import numpy_matrix, torch_matrix

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def h():
    import paper_2011_11188_b200 as s3

    assert torch.cuda.is_available(), "GPU tests need a B200"
    return s3.Handle(0)


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (200, 300, 100), (257, 129, 1000), (512, 768, 640),
                                   (1024, 1024, 1024)])
@pytest.mark.parametrize("kind", ["uniform", "loguni"])
def test_bf16x3_vs_oracle(h, orc, M, N, K, kind):
    A = numpy_matrix(kind, M, K, seed=M + 3)
    B = numpy_matrix(kind, K, N, seed=N + 4)
    C = h.sgemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), bf16x3=True).cpu().numpy()
    Cs = orc.sgemm_bf16x3(A, B)
    C64 = orc.gemm64(A, B)
    e_or = np.linalg.norm(C - Cs) / np.linalg.norm(Cs)
    e64rel = np.linalg.norm(C - C64) / np.linalg.norm(C64)
    assert e_or <= 1e-6 and e64rel <= 1e-6, (e_or, e64rel)


@pytest.mark.parametrize("transA,transB", [(0, 0), (1, 1)])
def test_bf16x3_transposes_bitwise(h, transA, transB):
    M, N, K = 300, 400, 500
    opA = numpy_matrix("uniform", M, K, seed=1)
    opB = numpy_matrix("uniform", K, N, seed=2)
    As = np.ascontiguousarray(opA.T) if transA else opA
    Bs = np.ascontiguousarray(opB.T) if transB else opB
    C = h.sgemm_ex(torch.from_numpy(As).cuda(), torch.from_numpy(Bs).cuda(), transA=bool(transA),
                   transB=bool(transB), bf16x3=True)
    ref = h.sgemm(torch.from_numpy(opA).cuda(), torch.from_numpy(opB).cuda(), bf16x3=True)
    assert torch.equal(C.view(torch.int32), ref.view(torch.int32))


def test_bf16x3_integer_exact(h):
    A = numpy_matrix("int2", 300, 4096, seed=1)
    B = numpy_matrix("int2", 4096, 200, seed=2)
    C = h.sgemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), bf16x3=True).cpu().numpy()
    assert np.array_equal(C, (A.astype(np.int64) @ B.astype(np.int64)).astype(np.float32))


def test_bf16x3_full_size_sampled(h, orc):
    n = 8192
    A = torch_matrix("uniform", n, n, seed=71, device="cuda")
    B = torch_matrix("uniform", n, n, seed=72, device="cuda")
    C = h.sgemm(A, B, bf16x3=True)
    rng = np.random.Generator(np.random.PCG64(5))
    rows = np.sort(rng.choice(n, 32, replace=False))
    cols = np.sort(rng.choice(n, 32, replace=False))
    An, Bn = A.cpu().numpy(), B.cpu().numpy()
    X = orc.split_bf16x3(An[rows])
    Y = orc.split_bf16x3(np.ascontiguousarray(Bn[:, cols]))
    Cs = orc.gemm_bf16x3_planes(X, Y)
    Cg = C[torch.from_numpy(rows).cuda()][:, torch.from_numpy(cols).cuda()].cpu().numpy()
    C64 = An[rows].astype(np.float64) @ Bn[:, cols].astype(np.float64)
    assert np.linalg.norm(Cg - Cs) / np.linalg.norm(Cs) <= 1e-6
    assert np.linalg.norm(Cg - C64) / np.linalg.norm(C64) <= 1e-6


@pytest.mark.parametrize("shape", [(1, 1), (65, 129), (300, 200), (1000, 72)])
@pytest.mark.parametrize("kind,scale", [("uniform", 1.0), ("loguni", 1.0), ("uniform", 1e-36), ("uniform", 1e36)])
def test_bf16x3_planes_bit_exact(h, orc, shape, kind, scale):
    rows, cols = shape
    X = (numpy_matrix(kind, rows, cols, seed=rows + cols) * np.float32(scale)).astype(np.float32)
    ref = orc.split_bf16x3(X)
    Xd = torch.from_numpy(X).cuda()
    for tr in (False, True):
        ps = h.split_bf16x3(Xd, transpose=tr)
        for p, r in zip(ps, ref):
            got = p.cpu().numpy().view(np.uint16)
            got = got[:cols, :rows].T if tr else got[:rows, :cols]
            assert np.array_equal(got, r)
