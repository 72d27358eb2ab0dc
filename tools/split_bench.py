"""Time the split-phase kernels alone at N x N (CUDA events, back to back): GB/s algorithmic."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2011_11188_b200 as s3  # noqa: E402
from workloads import torch_matrix  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
h = s3.Handle(0)
X = torch_matrix("uniform", n, n, seed=0)
d = torch.zeros(1, device="cuda")
h.maxabs(X, d)
hi, lo, sx = h.split(X, d)
hit, lot, _ = h.split(X, d, transpose=True)


def t(fn, reps=20):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


res = {"n": n,
       "maxabs_us": 1e3 * t(lambda: h.maxabs(X, d)),
       "split_us": 1e3 * t(lambda: h.split(X, d, hi=hi, lo=lo, d_sexp=sx)),
       "split_t_us": 1e3 * t(lambda: h.split(X, d, transpose=True, hi=hit, lo=lot, d_sexp=sx))}
b = n * n * 4
res["maxabs_GBs"] = b / (res["maxabs_us"] * 1e3)
res["split_GBs"] = 2 * b / (res["split_us"] * 1e3)
res["split_t_GBs"] = 2 * b / (res["split_t_us"] * 1e3)
print(json.dumps(res))
