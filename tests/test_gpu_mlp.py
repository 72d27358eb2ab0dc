"""NEXT #3: split-3 inside a dense-network training step (SPEC.md mlp, criteria 9-10).

GPU network (paper_2011_11188_b200.mlp, all GEMMs through split3_sgemm_ex) vs the fp64 reference
network (oracle/mlp.py, exact products) on the same seeded weights and batches.
"""
import math

import numpy as np
import pytest
import torch

from oracle import mlp as omlp
from workloads import make_blobs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def h():
    import paper_2011_11188_b200 as s3

    assert torch.cuda.is_available(), "GPU tests need a B200"
    return s3.Handle(0)


def _net(h, sizes, seed, mode="three"):
    from paper_2011_11188_b200.mlp import DenseNet

    return DenseNet(sizes, seed=seed, mode=mode, h=h)


def _np(ts):
    return [t.cpu().numpy().astype(np.float64) for t in ts]


def test_zero_net_uniform_softmax_and_ln_k(h):
    from paper_2011_11188_b200.mlp import DenseNet

    k = 7
    Ws = [torch.zeros((10, 32), device="cuda"), torch.zeros((32, k), device="cuda")]
    bs = [torch.zeros(32, device="cuda"), torch.zeros(k, device="cuda")]
    net = DenseNet.from_weights(Ws, bs, h=h)
    X, y = make_blobs(100, k, 10, 3.0, 0)
    Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
    P = net.predict_proba(Xd).cpu().numpy()
    assert np.allclose(P, 1.0 / k, atol=1e-7)
    assert abs(net.loss(Xd, yd) - math.log(k)) < 1e-6


@pytest.mark.parametrize("sizes", [(64, 256, 10), (300, 512, 512, 3)])
def test_forward_and_gradients_vs_fp64(h, sizes):
    """SPEC: 3-term forward within 1e-5 of exact (probabilities), logits 1e-4; gradients 1e-4 rel."""
    net = _net(h, sizes, seed=3)
    X, y = make_blobs(512, sizes[-1], sizes[0], 4.0, 5)
    Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
    Ws, bs = _np(net.W), _np(net.b)
    acts = omlp.forward(Ws, bs, X)
    L = net.forward(Xd)[-1].cpu().numpy()
    assert np.max(np.abs(L - acts[-1])) <= 1e-4 * max(1.0, np.max(np.abs(acts[-1])))
    P = net.predict_proba(Xd).cpu().numpy()
    assert np.max(np.abs(P - omlp.softmax(acts[-1]))) <= 1e-5
    assert np.max(np.abs(P.sum(axis=1) - 1.0)) <= 1e-6
    loss, dWs, dbs = net.backward(Xd, yd)
    assert abs(loss - omlp.loss(Ws, bs, X, y)) <= 1e-6 * max(1.0, abs(loss))
    rW, rb = omlp.backward(Ws, bs, X, y)
    for g, r in zip(_np(dWs) + _np(dbs), rW + rb):
        assert np.linalg.norm(g - r) <= 1e-4 * np.linalg.norm(r), np.linalg.norm(g - r) / np.linalg.norm(r)


def test_training_parity_blobs(h):
    """criterion 10: blobs (separation 6, 3 classes), 30 epochs: 3-term test accuracy within
    2 points of the fp64 network trained on the same batches; naive FP16 (1-term) as a control."""
    sizes = (20, 64, 3)
    X, y = make_blobs(1200, 3, 20, 6.0, 11)          # one draw of the clusters, split train/test
    Xtr, ytr, Xte, yte = X[:600], y[:600], X[600:], y[600:]
    lr, bsz = 0.5, 60
    batches = [(Xtr[i:i + bsz], ytr[i:i + bsz]) for e in range(30) for i in range(0, len(ytr), bsz)]
    res = {}
    for mode in ("three", "one"):
        net = _net(h, sizes, seed=21, mode=mode)
        W0, b0 = _np(net.W), _np(net.b)
        for X, y in batches:
            net.step(torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda(), lr)
        res[mode] = net.accuracy(torch.from_numpy(Xte).cuda(), torch.from_numpy(yte).cuda())
    Wr, br = omlp.sgd_train(W0, b0, batches, lr)
    ref_acc = float((omlp.forward(Wr, br, Xte)[-1].argmax(1) == yte).mean())
    print({"fp64": ref_acc, **res})
    assert abs(res["three"] - ref_acc) <= 0.02
    assert ref_acc > 0.9


def test_training_trajectory_close_to_fp64(h):
    """A few SGD steps on a wider net: 3-term weights stay within 1e-5 (relative) of fp64."""
    sizes = (128, 256, 10)
    X, y = make_blobs(256, 10, 128, 5.0, 31)
    net = _net(h, sizes, seed=32)
    W0, b0 = _np(net.W), _np(net.b)
    batches = [(X, y)] * 5
    for Xb, yb in batches:
        net.step(torch.from_numpy(Xb).cuda(), torch.from_numpy(yb).cuda(), 0.1)
    Wr, br = omlp.sgd_train(W0, b0, batches, 0.1)
    for w, r in zip(_np(net.W), Wr):
        assert np.linalg.norm(w - r) <= 1e-5 * np.linalg.norm(r)


def test_graph_captured_step_matches_eager(h):
    """The CUDA-graph training step produces the same weights as eager steps, bitwise."""
    from paper_2011_11188_b200.mlp import DenseNet

    sizes = (64, 128, 10)
    X, y = make_blobs(256, 10, 64, 5.0, 41)
    Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
    a = DenseNet(sizes, seed=5, h=h)
    b = DenseNet(sizes, seed=5, h=h)
    replay, loss = b.capture_step(Xd, yd, 0.05)   # capture performs one warm-up step
    a.step(Xd, yd, 0.05)
    for _ in range(4):
        a.step(Xd, yd, 0.05)
        replay()
    torch.cuda.synchronize()
    for wa, wb in zip(a.W + a.b, b.W + b.b):
        assert torch.equal(wa, wb)
