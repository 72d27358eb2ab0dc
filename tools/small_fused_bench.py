"""Small calls: the one-launch front end (prep2, separate split) vs fused B vs fused A (one GPU).

Eager split3_sgemm calls, median of --reps CUDA-event-timed calls after 5 warm-ups, 256 MiB L2
flush before each.  Writes gpurun_out/small_fused_bench.json.
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
p.add_argument("--reps", type=int, default=50)
p.add_argument("--shapes", default="64x64x64,512x512x512,1024x1024x1024,256x1024x1024,1024x256x1024,4096x256x256,"
                                   "256x4096x256,2048x2048x512,256x2048x2048,2048x256x2048,1024x1024x4096")
a = p.parse_args()
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")


def timed(fn, reps):
    for _ in range(5):
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


def handle(fa, fb):
    h = s3.Handle(0)
    h.set_fused_split_a(fa)
    h.set_fused_split(fb)
    return h


modes = {"prep": handle(0, 0), "fused_b": handle(0, 2), "fused_a": handle(2, 0), "default": s3.Handle(0)}
rows = []
for shp in a.shapes.split(","):
    M, N, K = (int(x) for x in shp.split("x"))
    A = torch_matrix("uniform", M, K, seed=1)
    B = torch_matrix("glorot", K, N, seed=2)
    C = torch.empty(M, N, device="cuda")
    r = {"M": M, "N": N, "K": K}
    for name, h in modes.items():
        r["us_" + name] = 1e3 * timed(lambda: h.sgemm(A, B, out=C), a.reps)
        r["launches_" + name] = h.last_launch_count()
    print(json.dumps(r), flush=True)
    rows.append(r)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(rows, open("gpurun_out/small_fused_bench.json", "w"), indent=1)
