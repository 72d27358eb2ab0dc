"""Small shapes through every entry point (for compute-sanitizer runs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2011_11188_b200 as s3  # noqa: E402
from workloads import torch_matrix  # noqa: E402

h = s3.Handle(0)
for (M, N, K) in ((300, 200, 500), (512, 512, 256), (1, 1, 1), (257, 129, 1000), (2048, 2560, 128)):
    A = torch_matrix("uniform", M, K, seed=1)
    B = torch_matrix("loguni", K, N, seed=2)
    for four, one in ((False, False), (True, False), (False, True)):
        h.sgemm(A, B, four_term=four, one_term=one)
    h.sgemm_ex(A.t().contiguous(), B, transA=True)
    P = h.presplit(B, role=1)
    h.sgemm_ex(A, P)
torch.cuda.synchronize()
print("ok")
