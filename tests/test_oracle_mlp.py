"""Pins of the fp64 reference network (oracle/mlp.py): SPEC.md criterion 9 and closed forms."""
import numpy as np

from oracle import mlp as omlp
from workloads import make_blobs


def _net(seed, sizes=(5, 7, 4)):
    rng = np.random.Generator(np.random.PCG64(seed))
    Ws = [rng.uniform(-1, 1, (a, b)) for a, b in zip(sizes[:-1], sizes[1:])]
    bs = [rng.uniform(-0.5, 0.5, b) for b in sizes[1:]]
    return Ws, bs


def test_gradients_vs_central_differences():
    """criterion 9: analytic backprop vs fp64 central differences (h = 1e-4) over 10 nets."""
    worst = 0.0
    for seed in range(10):
        Ws, bs = _net(seed)
        X, y = make_blobs(6, 4, 5, 3.0, seed)
        dWs, dbs = omlp.backward(Ws, bs, X, y)
        for params, grads in ((Ws, dWs), (bs, dbs)):
            for p, g in zip(params, grads):
                for idx in np.ndindex(p.shape):
                    old = p[idx]
                    p[idx] = old + 1e-4
                    lp = omlp.loss(Ws, bs, X, y)
                    p[idx] = old - 1e-4
                    lm = omlp.loss(Ws, bs, X, y)
                    p[idx] = old
                    fd = (lp - lm) / 2e-4
                    worst = max(worst, abs(fd - g[idx]) / max(1e-3, abs(fd), abs(g[idx])))
    assert worst < 1e-6, worst


def test_zero_net_closed_forms():
    k = 5
    Ws = [np.zeros((3, 6)), np.zeros((6, k))]
    bs = [np.zeros(6), np.zeros(k)]
    X, y = make_blobs(40, k, 3, 2.0, 1)
    assert abs(omlp.loss(Ws, bs, X, y) - np.log(k)) < 1e-15
    P = omlp.softmax(omlp.forward(Ws, bs, X)[-1])
    assert np.allclose(P, 1.0 / k)
    _, dbs = omlp.backward(Ws, bs, X, y)
    onehot_mean = np.bincount(y, minlength=k) / len(y)
    assert np.allclose(dbs[-1], 1.0 / k - onehot_mean)


def test_make_blobs_deterministic_and_separable():
    X1, y1 = make_blobs(300, 3, 10, 10.0, 7)
    X2, y2 = make_blobs(300, 3, 10, 10.0, 7)
    assert np.array_equal(X1, X2) and np.array_equal(y1, y2)
    # nearest-centroid classifier is perfect at separation 10
    cent = np.stack([X1[y1 == c].mean(0) for c in range(3)])
    pred = np.argmin(((X1[:, None, :] - cent[None]) ** 2).sum(-1), axis=1)
    assert (pred == y1).mean() > 0.99
