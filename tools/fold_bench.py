"""Folded accumulator (split3_set_fold) vs the D_hi / D_mid kernel, 3- and 4-term, whole calls
(median of --reps CUDA-event-timed calls after 3 warm-ups, 256 MiB L2 flush before each; modes
alternate per shape).  Writes gpurun_out/fold_bench.json."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2011_11188_b200 as s3  # noqa: E402
from workloads import torch_matrix  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--reps", type=int, default=30)
p.add_argument("--shapes", default="2048x2048x2048,4096x4096x1024,4096x4096x4096,8192x8192x2048,8192x8192x8192,"
                                   "4096x8192x8192,1024x8192x8192,256x8192x8192")
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


def handle(fold):
    h = s3.Handle(0)
    h.set_fold(fold)
    return h


modes = {"unfolded": handle(0), "folded": handle(2)}
rows = []
for shp in a.shapes.split(","):
    M, N, K = (int(x) for x in shp.split("x"))
    A = torch_matrix("uniform", M, K, seed=1)
    B = torch_matrix("uniform", K, N, seed=2)
    C = torch.empty(M, N, device="cuda")
    reps = a.reps if M * N * K <= 8192 ** 3 else 5
    r = {"M": M, "N": N, "K": K}
    for terms in (3, 4):
        for name, h in modes.items():
            r[f"ms_{name}_{terms}"] = timed(lambda: h.sgemm(A, B, out=C, four_term=terms == 4), reps)
        r[f"speedup_fold_{terms}"] = r[f"ms_unfolded_{terms}"] / r[f"ms_folded_{terms}"]
    print(json.dumps(r), flush=True)
    rows.append(r)
    del A, B, C
    torch.cuda.empty_cache()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(rows, open("gpurun_out/fold_bench.json", "w"), indent=1)
