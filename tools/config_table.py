"""Throughput of the whole split3_sgemm call for every BASELINE.json config (one GPU).

Times each configuration back to back for ~--secs seconds (CUDA events on the launching
stream, NVML clock samples), plus the GEMM kernel alone (library timing hook).  Writes
gpurun_out/config_table.json; tools/config_table.py --md turns it into a markdown table.
"""
import argparse
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

p = argparse.ArgumentParser()
p.add_argument("--secs", type=float, default=1.5)
p.add_argument("--md", default=None)
p.add_argument("--only", default=None)
a = p.parse_args()

if a.md:
    rows = json.load(open(a.md))
    print("| config | M | N | K | terms | ms / call | effective TFLOP/s (2MNK/t) | FP16 TFLOP/s (GEMM kernel) | GEMM share | SM MHz |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        print(f"| {r['config']} | {r['M']} | {r['N']} | {r['K']} | {r['terms']} | {r['ms']:.3f} | {r['eff_tflops']:.1f} | "
              f"{r['gemm_fp16_tflops']:.1f} | {r['gemm_share']:.0%} | {r['sm_mhz']:.0f} |")
    sys.exit(0)

import pynvml  # noqa: E402
import torch  # noqa: E402

import paper_2011_11188_b200 as s3  # noqa: E402
from workloads import torch_matrix  # noqa: E402

pynvml.nvmlInit()
nv = pynvml.nvmlDeviceGetHandleByIndex(0)
h = s3.Handle(0)
CONFIGS = [("D1 N=64", 64, 64, 64, "uniform", "uniform", 3)]
for n in (4096, 16384):
    for t in (3, 4):
        CONFIGS.append((f"D2 N={n}", n, n, n, "uniform", "uniform", t))
    CONFIGS.append((f"NEXT#4 bf16x3 N={n}", n, n, n, "uniform", "uniform", 6))
for M in (256, 1024, 4096):
    for KN in (1024, 4096, 8192):
        CONFIGS.append((f"D3 dense M={M}", M, KN, KN, "uniform", "glorot", 3))
        CONFIGS.append((f"D3 dense M={M}, W pre-split", M, KN, KN, "uniform", "glorot", 3))
CONFIGS.append(("D4 loguni N=8192", 8192, 8192, 8192, "loguni", "loguni", 3))
CONFIGS.append(("D5 N=65536 (1 GPU)", 65536, 65536, 65536, "uniform", "uniform", 3))
res = []
for name, M, N, K, ka, kb, terms in CONFIGS:
    if a.only and a.only not in name:
        continue
    A = torch_matrix(ka, M, K, seed=1, device="cuda")
    B = torch_matrix(kb, K, N, seed=2, device="cuda")
    C = torch.empty((M, N), device="cuda")
    four = terms == 4
    if "pre-split" in name:
        Wp = h.presplit(B, role=1)
        call = lambda: h.sgemm_ex(A, Wp, out=C)    # noqa: E731
    elif terms == 6:
        call = lambda: h.sgemm(A, B, out=C, bf16x3=True)   # noqa: E731
    else:
        call = lambda: h.sgemm(A, B, out=C, four_term=four)   # noqa: E731
    call()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    call()
    torch.cuda.synchronize()
    reps = max(3, min(2000, int(a.secs / max(time.perf_counter() - t0, 1e-5))))
    clk, stop = [], [False]

    def samp():
        while not stop[0]:
            clk.append(pynvml.nvmlDeviceGetClockInfo(nv, pynvml.NVML_CLOCK_SM))
            time.sleep(0.01)

    th = threading.Thread(target=samp, daemon=True)
    th.start()
    h.timing_enable(True)
    h.timing_read()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        call()
    e1.record()
    torch.cuda.synchronize()
    stop[0] = True
    th.join()
    h.timing_enable(False)
    split_ms, gemm_ms, n = h.timing_read()
    ms = e0.elapsed_time(e1) / reps
    r = {"config": name, "M": M, "N": N, "K": K, "terms": terms, "ms": ms, "reps": reps,
         "eff_tflops": 2.0 * M * N * K / (ms / 1e3) / 1e12,
         "gemm_fp16_tflops": terms * 2.0 * M * N * K / (gemm_ms / n / 1e3) / 1e12,
         "gemm_share": gemm_ms / n / ms, "split_ms": split_ms / n,
         "sm_mhz": float(sorted(clk)[len(clk) // 2]) if clk else float("nan")}
    print(json.dumps(r), flush=True)
    res.append(r)
    del A, B, C
    torch.cuda.empty_cache()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/config_table.json", "w"), indent=1)
