"""fp64 reference dense network (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

The same architecture as paper_2011_11188_b200/mlp.py (ReLU hidden layers, softmax output,
mean cross-entropy, SGD) with every operation in fp64 and exact matrix products ("Oracle64").
Pinned by central finite differences (tests/test_oracle_mlp.py; SPEC.md criterion 9).
"""
import numpy as np


def forward(Ws, bs, X):
    acts = [np.asarray(X, np.float64)]
    for i, (w, b) in enumerate(zip(Ws, bs)):
        z = acts[-1] @ np.asarray(w, np.float64) + np.asarray(b, np.float64)
        acts.append(np.maximum(z, 0.0) if i < len(Ws) - 1 else z)
    return acts


def softmax(L):
    L = L - L.max(axis=1, keepdims=True)
    e = np.exp(L)
    return e / e.sum(axis=1, keepdims=True)


def loss(Ws, bs, X, y):
    L = forward(Ws, bs, X)[-1]
    Lm = L - L.max(axis=1, keepdims=True)
    logp = Lm - np.log(np.exp(Lm).sum(axis=1, keepdims=True))
    return float(-logp[np.arange(len(y)), y].mean())


def backward(Ws, bs, X, y):
    acts = forward(Ws, bs, X)
    M = len(y)
    P = softmax(acts[-1])
    dZ = P.copy()
    dZ[np.arange(M), y] -= 1.0
    dZ /= M
    dWs, dbs = [None] * len(Ws), [None] * len(Ws)
    for i in range(len(Ws) - 1, -1, -1):
        dWs[i] = acts[i].T @ dZ
        dbs[i] = dZ.sum(axis=0)
        if i > 0:
            dH = dZ @ np.asarray(Ws[i], np.float64).T
            dZ = dH * (acts[i] > 0)
    return dWs, dbs


def sgd_train(Ws, bs, batches, lr):
    Ws = [np.asarray(w, np.float64).copy() for w in Ws]
    bs = [np.asarray(b, np.float64).copy() for b in bs]
    for X, y in batches:
        dWs, dbs = backward(Ws, bs, X, y)
        for w, g in zip(Ws, dWs):
            w -= lr * g
        for b, g in zip(bs, dbs):
            b -= lr * g
    return Ws, bs
