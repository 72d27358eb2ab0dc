"""Per-kernel breakdown of one split3_sgemm call (device durations via the torch profiler / CUPTI)
next to the call's own event-timed duration, so launch gaps between the kernels show up.

  python tools/call_breakdown.py 4096 8192 256x1024x1024 ...   (N or MxNxK)
"""
import json
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2011_11188_b200 as s3  # noqa: E402
from workloads import torch_matrix  # noqa: E402

h = s3.Handle(0)
flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")    # 256 MiB > L2
for arg in sys.argv[1:] or ["4096"]:
    M, N, K = (int(v) for v in arg.split("x")) if "x" in arg else (int(arg),) * 3
    n = arg
    A = torch_matrix("uniform", M, K, seed=0)
    B = torch_matrix("uniform", K, N, seed=1)
    C = torch.empty((M, N), device="cuda")
    for _ in range(5):
        h.sgemm(A, B, out=C)
    reps = 50
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * reps)]
    torch.cuda.synchronize()
    for i in range(reps):
        flush.zero_()
        ev[2 * i].record()
        h.sgemm(A, B, out=C)
        ev[2 * i + 1].record()
    torch.cuda.synchronize()
    call_ms = sorted(ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(reps))[reps // 2]
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            flush.zero_()
            h.sgemm(A, B, out=C)
        torch.cuda.synchronize()
    per = defaultdict(list)
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            per[e.name].append(e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total)
    kern = {k: sum(v) / reps / 1e3 for k, v in per.items() if "zero" not in k.lower() and "fill" not in k.lower()}
    tot = sum(kern.values())
    print(json.dumps({"n": n, "call_ms_median": call_ms, "kernels_ms_per_call": {k[:60]: round(v, 4) for k, v in kern.items()},
                      "sum_kernels_ms": round(tot, 4), "gaps_ms": round(call_ms - tot, 4),
                      "tflops_effective": 2.0 * M * N * K / (call_ms / 1e3) / 1e12}))
