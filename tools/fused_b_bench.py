"""Fused split of B (NEXT #2) vs the separate split pass vs a pre-split B, per shape (one GPU).

Whole split3_sgemm calls, median of --reps CUDA-event-timed calls after 3 warm-ups, a 256 MiB
L2 flush before each timed call.  Prints one JSON line per shape and writes
gpurun_out/fused_b_bench.json.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2011_11188_b200 as s3  # noqa: E402
from workloads import torch_matrix  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--reps", type=int, default=20)
p.add_argument("--shapes", default="256x1024x1024,256x4096x4096,256x8192x8192,1024x4096x4096,1024x8192x8192,"
                                   "2048x8192x8192,4096x4096x4096,4096x8192x8192,8192x8192x8192,16384x16384x16384")
p.add_argument("--transb", action="store_true", help="B given as B^T (stored N x K): the K-major fused path")
a = p.parse_args()

flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")


def timed(fn, reps):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


hs, hf = s3.Handle(0), s3.Handle(0)
hs.set_fused_split(0)
hf.set_fused_split(2)
hs.set_fused_split_a(0)      # B's fusion alone (no fused-A auto choice for N < M)
hf.set_fused_split_a(0)
rows = []
for shp in a.shapes.split(","):
    M, N, K = (int(x) for x in shp.split("x"))
    A = torch_matrix("uniform", M, K, seed=1)
    tb = a.transb
    B = torch_matrix("glorot", N, K, seed=2) if tb else torch_matrix("glorot", K, N, seed=2)
    C = torch.empty(M, N, device="cuda")
    reps = a.reps if M * N * K <= 8192 ** 3 else 5
    t_sep = timed(lambda: hs.sgemm_ex(A, B, transB=tb, out=C), reps)
    Cs = C.clone()
    t_fus = timed(lambda: hf.sgemm_ex(A, B, transB=tb, out=C), reps)
    same = bool(torch.equal(C.view(torch.int32), Cs.view(torch.int32)))
    Bp = hs.presplit_stored(B)
    t_pre = timed(lambda: hs.sgemm_ex(A, Bp, transB=tb, out=C), reps)
    fl = 2.0 * M * N * K
    r = {"M": M, "N": N, "K": K, "transB": tb, "ms_separate": t_sep, "ms_fused": t_fus, "ms_presplit_b": t_pre,
         "eff_tflops_separate": fl / t_sep / 1e9, "eff_tflops_fused": fl / t_fus / 1e9,
         "eff_tflops_presplit_b": fl / t_pre / 1e9, "speedup_fused": t_sep / t_fus, "bitwise_equal": same}
    print(json.dumps(r), flush=True)
    rows.append(r)
    del A, B, C, Cs, Bp
    torch.cuda.empty_cache()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(rows, open("gpurun_out/fused_b_bench%s.json" % ("_transb" if a.transb else ""), "w"), indent=1)
