"""split3_presplit_stored: the plain split of a stored matrix, reused as A or B with either
transpose (split3_matrix.stored = 1).  Same plane values and scale as splitting inside the call,
and the GEMM reads them with the same layouts -> C bitwise equal to the fp32-operand path."""
import pytest
import torch

import paper_2011_11188_b200 as s3
from paper_2011_11188_b200.mlp import DenseNet
from workloads import torch_matrix

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def h():
    return s3.Handle(0)


def _bits(C):
    return C.contiguous().view(torch.int32)


@pytest.mark.parametrize("transA,transB", [(0, 0), (1, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("kw", [{}, {"four_term": True}, {"one_term": True}])
@pytest.mark.parametrize("M,N,K", [(300, 200, 500), (1000, 1030, 129), (2048, 1536, 1024)])
def test_stored_planes_equal_fp32_path(h, transA, transB, kw, M, N, K):
    A = torch_matrix("uniform", K if transA else M, M if transA else K, seed=61)
    B = torch_matrix("loguni", N if transB else K, K if transB else N, seed=62)
    ref = h.sgemm_ex(A, B, transA=bool(transA), transB=bool(transB), **kw).clone()
    PA, PB = h.presplit_stored(A), h.presplit_stored(B)
    for a, b in [(PA, PB), (PA, B), (A, PB)]:
        C = h.sgemm_ex(a, b, transA=bool(transA), transB=bool(transB), **kw)
        assert torch.equal(_bits(C), _bits(ref))


def test_one_split_serves_both_roles(h):
    """W split once: X*W (W as B, MN-major) and dZ*W^T (W as B^T, K-major) and W^T*Y (W as A^T)."""
    W = torch_matrix("glorot", 768, 512, seed=63)
    X = torch_matrix("uniform", 256, 768, seed=64)
    dZ = torch_matrix("uniform", 256, 512, seed=65)
    Y = torch_matrix("uniform", 768, 128, seed=66)
    P = h.presplit_stored(W)
    assert torch.equal(_bits(h.sgemm_ex(X, P)), _bits(h.sgemm_ex(X, W)))
    assert torch.equal(_bits(h.sgemm_ex(dZ, P, transB=True)), _bits(h.sgemm_ex(dZ, W, transB=True)))
    assert torch.equal(_bits(h.sgemm_ex(P, Y, transA=True)), _bits(h.sgemm_ex(W, Y, transA=True)))


def test_stored_planes_bad_ldp(h):
    W = torch_matrix("uniform", 64, 100, seed=67)
    P = h.presplit_stored(W)
    P.hi, P.lo = P.hi[:, :96], P.lo[:, :96]       # a view whose row stride is still 104 ...
    bad = s3.split3.Planes(P.hi.contiguous(), P.lo.contiguous(), P.sexp, None, 64, 100, stored=True)
    with pytest.raises(s3.Split3Error):           # ... contiguous copy: ldp 96 < 100 columns
        h.sgemm_ex(torch_matrix("uniform", 8, 64, seed=68), bad)


def _old_backward(net, X, y):
    """The previous formulation: every GEMM gets fp32 operands (split inside each call)."""
    h = net.h
    acts = [X]
    for i, (w, b) in enumerate(zip(net.W, net.b)):
        Z = h.sgemm_ex(acts[-1], w)
        acts.append(h.bias_act(Z, b, relu=i < len(net.W) - 1, out=Z))
    _, dZ, loss = h.softmax_xent(acts[-1], y, want_probs=False, want_grad=True)
    dWs, dbs = [None] * len(net.W), [None] * len(net.W)
    for i in range(len(net.W) - 1, -1, -1):
        dWs[i] = h.sgemm_ex(acts[i], dZ, transA=True)
        dbs[i] = h.bias_grad(dZ)
        if i > 0:
            dH = h.sgemm_ex(dZ, net.W[i], transB=True)
            dZ = h.relu_backward(dH, acts[i], out=dH)
    return loss, dWs, dbs


def test_dense_step_reuses_splits_bitwise(h):
    net = DenseNet([384, 512, 256, 10], seed=3, h=h)
    X = torch_matrix("uniform", 200, 384, seed=69)
    y = torch.randint(0, 10, (200,), device="cuda", dtype=torch.int32)
    loss_n, dW_n, db_n = net.backward_device(X, y)
    loss_o, dW_o, db_o = _old_backward(net, X, y)
    assert float(loss_n) == float(loss_o)
    for a, b in zip(dW_n + db_n, dW_o + db_o):
        assert torch.equal(_bits(a), _bits(b))
