"""Same-box library baselines (context for the roofline): cuBLAS via torch.matmul at N x N.

fp16 / bf16 inputs with FP32 accumulation (the practical tensor-core ceiling for the split-3
contraction), fp32 SGEMM (TF32 off) and TF32.  Each is run back to back for --secs seconds
(sustained, power-capped) with NVML clock sampling.  Output: JSON lines + gpurun_out/baselines.json.
"""
import argparse
import json
import os
import threading
import time

import pynvml
import torch

p = argparse.ArgumentParser()
p.add_argument("--n", type=int, default=16384)
p.add_argument("--secs", type=float, default=4.0)
a = p.parse_args()
pynvml.nvmlInit()
nv = pynvml.nvmlDeviceGetHandleByIndex(0)
n = a.n
res = []
for name, dt, tf32 in (("fp16", torch.float16, False), ("bf16", torch.bfloat16, False),
                       ("tf32", torch.float32, True), ("fp32", torch.float32, False)):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    torch.backends.cuda.matmul.allow_fp16_reduced_precision_reduction = False
    torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = False
    A = torch.rand((n, n), device="cuda").to(dt)
    B = torch.rand((n, n), device="cuda").to(dt)
    C = torch.matmul(A, B)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    torch.matmul(A, B, out=C)
    torch.cuda.synchronize()
    one = time.perf_counter() - t0
    reps = max(3, int(a.secs / one))
    clk, pw, stop = [], [], [False]

    def samp():
        while not stop[0]:
            clk.append(pynvml.nvmlDeviceGetClockInfo(nv, pynvml.NVML_CLOCK_SM))
            pw.append(pynvml.nvmlDeviceGetPowerUsage(nv) / 1000)
            time.sleep(0.01)

    th = threading.Thread(target=samp, daemon=True)
    th.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        torch.matmul(A, B, out=C)
    e1.record()
    torch.cuda.synchronize()
    stop[0] = True
    th.join()
    ms = e0.elapsed_time(e1) / reps
    tf = 2.0 * n ** 3 / (ms / 1e3) / 1e12
    mhz = sorted(clk)[len(clk) // 2]
    r = {"lib": "cuBLAS (torch.matmul)", "dtype": name, "n": n, "ms": round(ms, 3), "tflops": round(tf, 1),
         "sm_mhz_median": mhz, "watts_max": round(max(pw)), "per_clock_eff_vs_8192flop": round(
             tf * 1e12 / (148 * 8192 * mhz * 1e6) * (1 if name in ("fp16", "bf16") else 2), 3), "reps": reps}
    print(json.dumps(r), flush=True)
    res.append(r)
    del A, B, C
    torch.cuda.empty_cache()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/baselines.json", "w"), indent=1)
