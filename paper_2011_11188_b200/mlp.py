"""Dense network trained with split-FP16 GEMMs.

"the form of operations in DNN are theoretically able to well approximate operations of fp32
using mixed-precision operations in fp16".  Every matrix product of the step —
forward Z = H W, backward dW = H^T dZ and dH = dZ W^T — runs through split3_sgemm_ex (3 FP16
tensor-core products, or 4 / 1 as controls); bias, ReLU, softmax cross-entropy, bias gradients
and the SGD update are the library's FP32 kernels (SPEC.md mlp ledger: only GEMMs in reduced
precision).  Architecture: ReLU hidden layers, softmax output, mean cross-entropy.
"""
from __future__ import annotations

import math

import numpy as np
import torch

from .split3 import Handle, handle

MODES = {"three": {}, "four": {"four_term": True}, "one": {"one_term": True}}


class DenseNet:
    def __init__(self, sizes, seed: int = 0, mode: str = "three", device="cuda", h: Handle | None = None):
        if mode not in MODES:
            raise ValueError(f"mode must be one of {sorted(MODES)}")
        self.sizes = list(sizes)
        self.mode = mode
        self.h = h or handle(torch.device(device))
        rng = np.random.Generator(np.random.PCG64(seed))
        self.W, self.b = [], []
        for fin, fout in zip(self.sizes[:-1], self.sizes[1:]):
            lim = math.sqrt(6.0 / (fin + fout))   # Glorot uniform (SPEC.md mlp ledger)
            w = ((2.0 * rng.random((fin, fout)) - 1.0) * lim).astype(np.float32)
            self.W.append(torch.from_numpy(w).to(device))
            self.b.append(torch.zeros(fout, dtype=torch.float32, device=device))

    @classmethod
    def from_weights(cls, Ws, bs, mode="three", h=None):
        net = cls.__new__(cls)
        net.sizes = [Ws[0].shape[0]] + [w.shape[1] for w in Ws]
        net.mode = mode
        net.h = h or handle(Ws[0].device)
        net.W = [w.contiguous() for w in Ws]
        net.b = [b.contiguous() for b in bs]
        return net

    def _mm(self, A, B, transA=False, transB=False):
        return self.h.sgemm_ex(A, B, transA=transA, transB=transB, **MODES[self.mode])

    # matrices at least this large are split once per step and reused; smaller ones go to the GEMMs
    # as fp32 (an eager small net is host-bound: a separate split is one more call per matrix)
    REUSE_MIN_ELEMS = 4 << 20

    def _split(self, X):
        """The plain split of a stored matrix (split3_presplit_stored), reused by every GEMM that
        reads X in the step: W in X*W and dZ*W^T, H in H*W and H^T*dZ, dZ in H^T*dZ and dZ*W^T.
        Same planes and scale as splitting inside each call -> bitwise the same products, so small
        matrices in eager mode are simply passed as fp32 (split inside each GEMM call)."""
        if X.numel() >= self.REUSE_MIN_ELEMS or torch.cuda.is_current_stream_capturing():
            return self.h.presplit_stored(X)
        return X

    def _forward(self, X):
        """(activations [X, H1, ..., logits], planes of [X, H1, ...], planes of the weights)."""
        acts, act_planes, w_planes = [X], [], []
        L = len(self.W)
        for i, (w, b) in enumerate(zip(self.W, self.b)):
            act_planes.append(self._split(acts[-1]))
            w_planes.append(self._split(w))
            Z = self._mm(act_planes[-1], w_planes[-1])
            acts.append(self.h.bias_act(Z, b, relu=i < L - 1, out=Z))
        return acts, act_planes, w_planes

    def forward(self, X):
        """Per-layer activations [X, H1, ..., logits] (logits before softmax)."""
        return self._forward(X)[0]

    def predict_proba(self, X):
        P, _, _ = self.h.softmax_xent(self.forward(X)[-1], None, want_probs=True, want_grad=False)
        return P

    def loss(self, X, y):
        _, _, loss = self.h.softmax_xent(self.forward(X)[-1], y, want_probs=False, want_grad=False)
        return float(loss)

    def backward(self, X, y):
        """(loss, [dW], [db]) of the mean softmax cross-entropy."""
        loss, dWs, dbs = self.backward_device(X, y)
        return float(loss), dWs, dbs

    def backward_device(self, X, y):
        """As backward(), with the loss left on the device (no host synchronisation)."""
        acts, act_planes, w_planes = self._forward(X)
        _, dZ, loss = self.h.softmax_xent(acts[-1], y, want_probs=False, want_grad=True)
        dWs, dbs = [None] * len(self.W), [None] * len(self.W)
        for i in range(len(self.W) - 1, -1, -1):
            dZp = self._split(dZ)
            dWs[i] = self._mm(act_planes[i], dZp, transA=True)     # H^T dZ
            dbs[i] = self.h.bias_grad(dZ)
            if i > 0:
                dH = self._mm(dZp, w_planes[i], transB=True)       # dZ W^T
                dZ = self.h.relu_backward(dH, acts[i], out=dH)
        return loss, dWs, dbs

    def step_device(self, X, y, lr: float):
        """One SGD step; returns the loss as a 0-d device tensor (capturable in a CUDA graph)."""
        loss, dWs, dbs = self.backward_device(X, y)
        for w, g in zip(self.W, dWs):
            self.h.sgd_update(w, g, lr)
        for b, g in zip(self.b, dbs):
            self.h.sgd_update(b, g, lr)
        return loss

    def step(self, X, y, lr: float):
        return float(self.step_device(X, y, lr))

    def capture_step(self, X, y, lr: float):
        """CUDA-graph the training step on the static batch buffers X, y (refill them in place
        between replays).  Returns (replay, loss_tensor)."""
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):          # warm-up on the capture stream: its handle + workspace
            self.step_device(X, y, lr)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                loss = self.step_device(X, y, lr)
        torch.cuda.current_stream().wait_stream(s)
        return g.replay, loss

    def accuracy(self, X, y):
        return float((self.forward(X)[-1].argmax(dim=1) == y).float().mean())
