"""Randomised shapes / flags / transposes / leading dimensions / offsets vs the oracle."""
import numpy as np
import pytest
import torch

from workloads import numpy_matrix

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def h():
    import paper_2011_11188_b200 as s3

    assert torch.cuda.is_available(), "GPU tests need a B200"
    return s3.Handle(0)


def _embed(X, pad_cols, off):
    """X stored inside a larger row-major buffer (leading dimension cols + pad, column offset)."""
    rows, cols = X.shape
    big = np.full((rows, cols + pad_cols + off), np.float32(7.0), np.float32)
    big[:, off:off + cols] = X
    t = torch.from_numpy(big).cuda()
    return t[:, off:off + cols]


@pytest.mark.parametrize("seed", range(24))
def test_fuzz(h, orc, seed):
    rng = np.random.Generator(np.random.PCG64(1000 + seed))
    M, N, K = (int(rng.integers(1, 1400)) for _ in range(3))
    mode = ["three", "four", "one", "bf16x3"][seed % 4]
    transA, transB = bool(rng.integers(0, 2)), bool(rng.integers(0, 2))
    kind = ["uniform", "loguni", "glorot"][int(rng.integers(0, 3))]
    opA = numpy_matrix(kind, M, K, seed=seed)
    opB = numpy_matrix(kind, K, N, seed=seed + 500)
    As = np.ascontiguousarray(opA.T) if transA else opA
    Bs = np.ascontiguousarray(opB.T) if transB else opB
    Ad = _embed(As, int(rng.integers(0, 9)), int(rng.integers(0, 3)))
    Bd = _embed(Bs, int(rng.integers(0, 9)), int(rng.integers(0, 3)))
    Cbig = torch.full((M, N + 5), 3.0, device="cuda")
    C = Cbig[:, 1:1 + N]
    kw = {"four_term": mode == "four", "one_term": mode == "one", "bf16x3": mode == "bf16x3"}
    h.sgemm_ex(Ad, Bd, transA=transA, transB=transB, out=C, **kw)
    Cn = C.cpu().numpy().astype(np.float64)
    if mode == "bf16x3":
        Cs = orc.sgemm_bf16x3(opA, opB)
    else:
        Cs = orc.sgemm(opA, opB, terms={"three": 3, "four": 4, "one": 1}[mode])
    den = np.linalg.norm(Cs)
    e_or = np.linalg.norm(Cn - Cs) / den if den > 0 else np.linalg.norm(Cn)
    assert e_or <= 1e-6, (M, N, K, mode, transA, transB, kind, e_or)
    cb = Cbig.cpu().numpy()
    assert np.all(cb[:, 0] == 3.0) and np.all(cb[:, N + 1:] == 3.0)
