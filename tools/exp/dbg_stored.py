import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2011_11188_b200 as s3
from workloads import torch_matrix
h = s3.Handle(0)
M, N, K = 300, 200, 500
A = torch_matrix("uniform", M, K, seed=61); B = torch_matrix("loguni", K, N, seed=62)
ref = h.sgemm_ex(A, B).clone()
PA, PB = h.presplit_stored(A), h.presplit_stored(B)
torch.cuda.synchronize()
# compare planes with the library's own split3_split
d = torch.zeros(1, device="cuda"); h.maxabs(A, d); hi, lo, sx = h.split(A, d)
print("A planes equal:", torch.equal(PA.hi[:, :K], hi[:, :K]), torch.equal(PA.lo[:, :K], lo[:, :K]), int(PA.sexp), int(sx))
d2 = torch.zeros(1, device="cuda"); h.maxabs(B, d2); hib, lob, sxb = h.split(B, d2)
print("B planes equal:", torch.equal(PB.hi[:, :N], hib[:, :N]), torch.equal(PB.lo[:, :N], lob[:, :N]), int(PB.sexp), int(sxb))
for name, (a, b) in {"PA,PB": (PA, PB), "PA,B": (PA, B), "A,PB": (A, PB)}.items():
    C = h.sgemm_ex(a, b)
    diff = (C - ref).abs().max().item()
    print(name, "max diff", diff, "rel", diff / ref.abs().max().item(), "nan", torch.isnan(C).any().item())
