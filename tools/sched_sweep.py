"""GEMM schedule sweep at N = 16384 (one GPU): raster group height (pair m-blocks) and L2 eviction
policies of the plane loads.  Each setting runs back to back for --secs seconds (power-capped clocks
settle) and reports the GEMM-kernel FP16 TFLOP/s (library timing hook) and the NVML SM clock.
Results never change a bit (tests/test_gpu_parity.py); this is for speed only."""
import argparse
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml  # noqa: E402
import torch  # noqa: E402

import paper_2011_11188_b200 as s3  # noqa: E402
from workloads import torch_matrix  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--n", type=int, default=16384)
p.add_argument("--secs", type=float, default=3.0)
p.add_argument("--groups", default="2,4,8,16,32")
p.add_argument("--pols", default="0:0,2:0,0:2,1:2")
a = p.parse_args()
pynvml.nvmlInit()
nv = pynvml.nvmlDeviceGetHandleByIndex(0)
n = a.n
h = s3.Handle(0)
A = torch_matrix("uniform", n, n, seed=0)
B = torch_matrix("uniform", n, n, seed=1)
C = torch.empty((n, n), device="cuda")
rows = []


def run(tag):
    for _ in range(2):
        h.sgemm(A, B, out=C)
    torch.cuda.synchronize()
    clocks, stop = [], [False]

    def poll():
        while not stop[0]:
            clocks.append(pynvml.nvmlDeviceGetClockInfo(nv, pynvml.NVML_CLOCK_SM))
            time.sleep(0.02)
    th = threading.Thread(target=poll)
    th.start()
    h.timing_enable(True)
    h.timing_read()
    t0 = time.time()
    k = 0
    while time.time() - t0 < a.secs:
        h.sgemm(A, B, out=C)
        k += 1
        if k % 8 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    stop[0] = True
    th.join()
    _, gm, nc = h.timing_read()
    h.timing_enable(False)
    clocks.sort()
    r = {"tag": tag, "gemm_ms": gm / nc, "fp16_tflops": 6.0 * n ** 3 / (gm / nc / 1e3) / 1e12,
         "sm_mhz_median": clocks[len(clocks) // 2] if clocks else None, "calls": nc}
    r["tflops_per_ghz"] = r["fp16_tflops"] / (r["sm_mhz_median"] / 1e3) if r["sm_mhz_median"] else None
    print(json.dumps(r), flush=True)
    rows.append(r)


for g in (int(x) for x in a.groups.split(",")):
    h.set_schedule(g, 0, 0)
    run(f"group_m={g}")
for pol in a.pols.split(","):
    pa, pb = (int(x) for x in pol.split(":"))
    h.set_schedule(0, pa, pb)
    run(f"pol_a={pa},pol_b={pb}")
run("default (again)")
os.makedirs("gpurun_out", exist_ok=True)
json.dump(rows, open("gpurun_out/sched_sweep.json", "w"), indent=1)
