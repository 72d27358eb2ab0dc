"""Run split3_sgemm a few times at one size (for ncu / sanitizer captures)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2011_11188_b200 as s3  # noqa: E402
from workloads import torch_matrix  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--n", type=int, default=8192)
p.add_argument("--m", type=int, default=0)
p.add_argument("--k", type=int, default=0)
p.add_argument("--reps", type=int, default=3)
p.add_argument("--terms", type=int, default=3)
a = p.parse_args()
M = a.m or a.n
K = a.k or a.n
A = torch_matrix("uniform", M, K, seed=0)
B = torch_matrix("uniform", K, a.n, seed=1)
h = s3.Handle(0)
for _ in range(a.reps):
    C = h.sgemm(A, B, four_term=a.terms == 4, one_term=a.terms == 1, bf16x3=a.terms == 6)
torch.cuda.synchronize()
print("ok", float(C[0, 0]))
