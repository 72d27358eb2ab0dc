"""Run the fused-A path (C^T = B^T A^T, transposed epilogue store) at one shape (ncu captures)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2011_11188_b200 as s3  # noqa: E402
from workloads import torch_matrix  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--m", type=int, default=8192)
p.add_argument("--n", type=int, default=1024)
p.add_argument("--k", type=int, default=8192)
p.add_argument("--reps", type=int, default=3)
a = p.parse_args()
A = torch_matrix("uniform", a.m, a.k, seed=0)
B = torch_matrix("glorot", a.k, a.n, seed=1)
h = s3.Handle(0)
h.set_fused_split_a(2)
for _ in range(a.reps):
    C = h.sgemm(A, B)
torch.cuda.synchronize()
assert h.last_path() & 2, h.last_path()
print("ok", float(C[0, 0]))
