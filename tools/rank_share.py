"""Config D5 at P GPUs, compute share of one rank, measured on ONE GPU (a projection, not the
multi-GPU metric: one GPU is all this run has).  For the pr x pc grid of dist.py, rank (0, 0)
splits its own A block ((N/P) x N) and B block (N x (N/P)) and, once the plane panels are
gathered, runs P GEMM pieces of (N/P) x (N/P) x N on whole tiles.  Timed with CUDA events:
the local split and the pieces at full width, and the pieces on 132 SMs (the budget the driver
gives pieces that overlap a gather).  Projected speedup = t(1 GPU, the whole N^3 call) / t(rank),
i.e. assuming the plane all-gathers (N^2 * 4 B / 2 inbound per rank) hide under the
GEMMs.  Writes gpurun_out/rank_share.json."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2011_11188_b200 as s3  # noqa: E402
from paper_2011_11188_b200.dist import grid_for  # noqa: E402
from workloads import torch_matrix  # noqa: E402

N = int(os.environ.get("RS_N", "65536"))
t1_ms = float(os.environ.get("RS_T1_MS", "0"))     # the 1-GPU whole call (config table D5), if known
res = {"N": N, "t1_ms": t1_ms, "cases": {}}
h = s3.Handle(0)
h.set_split_k(False)
for P in (2, 4, 8):
    pr, pc = grid_for(P)
    nb = N // P
    A = torch_matrix("uniform", nb, N, seed=1)          # own A block (K-major planes)
    B = torch_matrix("uniform", N, nb, seed=2)          # own B block (MN-major planes)
    d = torch.zeros(2, dtype=torch.float32, device="cuda")
    C = torch.empty((nb, nb), device="cuda")

    def split():
        h.maxabs(A, d[0:1])
        h.maxabs(B, d[1:2])
        return h.split(A, d[0:1], transpose=False), h.split(B, d[1:2], transpose=False)

    (a1, a2, sa), (b1, b2, sb) = split()
    pa = s3.split3.Planes(a1, a2, sa, None, nb, N, stored=True)
    pb = s3.split3.Planes(b1, b2, sb, None, N, nb, stored=True)

    def pieces(cap):
        h.set_max_sms(cap)
        for _ in range(P):
            h.sgemm_ex(pa, pb, out=C)
        h.set_max_sms(0)

    def timed(fn, reps=2):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    t_split = timed(split, 3)
    t_full = timed(lambda: pieces(0), 1)
    t_cap = timed(lambda: pieces(132), 1)
    case = {"grid": [pr, pc], "piece": [nb, nb, N], "pieces": P, "split_ms": t_split, "gemm_full_ms": t_full,
            "gemm_132sms_ms": t_cap, "rank_ms_full": t_split + t_full, "rank_ms_132sms": t_split + t_cap,
            "gather_bytes_inbound": N * N * 4 // 2 - (nb * N * 4)}
    flops = 2.0 * N ** 3
    case["projected_effective_tflops_full"] = flops / ((t_split + t_full) / 1e3) / 1e12
    case["projected_effective_tflops_132sms"] = flops / ((t_split + t_cap) / 1e3) / 1e12
    if t1_ms:
        case["projected_speedup_full"] = t1_ms / (t_split + t_full)
        case["projected_speedup_132sms"] = t1_ms / (t_split + t_cap)
    res["cases"][str(P)] = case
    print(json.dumps(case), flush=True)
    del A, B, C, pa, pb, a1, a2, b1, b2
    torch.cuda.empty_cache()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/rank_share.json", "w"), indent=1)
