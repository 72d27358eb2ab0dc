"""Fused split of A (NEXT #2, the transposed problem C^T = B^T A^T) vs the separate split vs fused B
vs the default choice, per shape (one GPU).

Whole split3_sgemm calls, median of --reps CUDA-event-timed calls after 3 warm-ups, a 256 MiB L2
flush before each timed call.  Prints one JSON line per shape and writes
gpurun_out/fused_a_bench.json.
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
p.add_argument("--shapes", default="4096x256x4096,8192x256x8192,4096x1024x1024,4096x1024x4096,8192x1024x8192,"
                                   "8192x2048x8192,4096x4096x1024,16384x4096x4096,4096x256x256,1024x256x1024")
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


def handle(fa, fb):
    h = s3.Handle(0)
    h.set_fused_split_a(fa)
    h.set_fused_split(fb)
    return h


modes = {"separate": handle(0, 0), "fused_a": handle(2, 0), "fused_b": handle(0, 2), "default": s3.Handle(0),
         "auto": handle(1, 1)}
rows = []
for shp in a.shapes.split(","):
    M, N, K = (int(x) for x in shp.split("x"))
    A = torch_matrix("uniform", M, K, seed=1)
    B = torch_matrix("glorot", K, N, seed=2)
    C = torch.empty(M, N, device="cuda")
    reps = a.reps if M * N * K <= 8192 ** 3 else 5
    r = {"M": M, "N": N, "K": K}
    ref = None
    for name, h in modes.items():
        r["ms_" + name] = timed(lambda: h.sgemm(A, B, out=C), reps)
        r["launches_" + name] = h.last_launch_count()
        if ref is None:
            ref = C.clone()
        else:
            r["bitwise_" + name] = bool(torch.equal(C.view(torch.int32), ref.view(torch.int32)))
    Ap = modes["separate"].presplit(A, role=0)
    r["ms_presplit_a"] = timed(lambda: modes["separate"].sgemm_ex(Ap, B, out=C), reps)
    fl = 2.0 * M * N * K
    for k in list(r):
        if k.startswith("ms_"):
            r["eff_tflops_" + k[3:]] = fl / r[k] / 1e9
    r["speedup_fused_a"] = r["ms_separate"] / r["ms_fused_a"]
    print(json.dumps(r), flush=True)
    rows.append(r)
    del A, B, C, ref, Ap
    torch.cuda.empty_cache()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(rows, open("gpurun_out/fused_a_bench.json", "w"), indent=1)
