"""Time the GEMM kernel alone (split3_gemm_planes) over promotion periods / terms / sizes."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2011_11188_b200 as s3  # noqa: E402
from workloads import torch_matrix  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--sizes", default="8192,16384")
p.add_argument("--promos", default="1,2,4,8,1024")
p.add_argument("--terms", default="3,1")
p.add_argument("--reps", type=int, default=10)
p.add_argument("--secs", type=float, default=0.6)
p.add_argument("--wave", default="1")
p.add_argument("--sched", default="0:0:0", help="comma list of group_m:polA:polB")
a = p.parse_args()

import threading  # noqa: E402

import pynvml  # noqa: E402

pynvml.nvmlInit()
_nv = pynvml.nvmlDeviceGetHandleByIndex(int(os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0] or 0))


class Clk:
    def __enter__(self):
        self.v, self.p, self.stop = [], [], False
        self.t = threading.Thread(target=self.run, daemon=True)
        self.t.start()
        return self

    def run(self):
        while not self.stop:
            self.v.append(pynvml.nvmlDeviceGetClockInfo(_nv, pynvml.NVML_CLOCK_SM))
            self.p.append(pynvml.nvmlDeviceGetPowerUsage(_nv) / 1000.0)
            time.sleep(0.01)

    def __exit__(self, *a):
        self.stop = True
        self.t.join()


import time  # noqa: E402
h = s3.Handle(0)
res = []
for n in [int(x) for x in a.sizes.split(",")]:
    A = torch_matrix("uniform", n, n, seed=0)
    B = torch_matrix("uniform", n, n, seed=1)
    dmax = torch.zeros(2, dtype=torch.float32, device="cuda")
    h.maxabs(A, dmax[0:1]); h.maxabs(B, dmax[1:2])
    A1, A2, sA = h.split(A, dmax[0:1])
    B1, B2, sB = h.split(B, dmax[1:2], transpose=True)
    del A, B
    C = torch.empty((n, n), device="cuda")
    for terms in [int(x) for x in a.terms.split(",")]:
        for pr, wv, sc in [(int(x), int(w), c) for x in a.promos.split(",") for w in a.wave.split(",")
                           for c in a.sched.split(",")]:
            h.set_promotion(pr)
            h.set_wave_sync(bool(wv))
            h.set_schedule(*[int(v) for v in sc.split(":")])
            for _ in range(2):
                h.gemm_planes(n, n, n, A1, A2, sA, B1, B2, sB, out=C, four_term=terms == 4, one_term=terms == 1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            h.gemm_planes(n, n, n, A1, A2, sA, B1, B2, sB, out=C, four_term=terms == 4, one_term=terms == 1)
            torch.cuda.synchronize()
            reps = max(a.reps, int(a.secs / max(time.perf_counter() - t0, 1e-4)))
            with Clk() as ck:
                e0.record()
                for _ in range(reps):
                    h.gemm_planes(n, n, n, A1, A2, sA, B1, B2, sB, out=C, four_term=terms == 4, one_term=terms == 1)
                e1.record()
                torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            tf = terms * 2.0 * n ** 3 / (ms / 1e3) / 1e12
            mhz = float(sorted(ck.v)[len(ck.v) // 2]) if ck.v else float("nan")
            r = {"n": n, "terms": terms, "promo": pr, "wave": wv, "sched": sc, "ms": round(ms, 3), "fp16_tflops": round(tf, 1),
                 "eff_tflops": round(2.0 * n ** 3 / (ms / 1e3) / 1e12, 1), "sm_mhz": mhz,
                 "watts": round(max(ck.p), 0) if ck.p else None,
                 "per_clock_eff": round(tf * 1e12 / (148 * 8192 * mhz * 1e6), 3)}
            print(json.dumps(r), flush=True)
            res.append(r)
h.set_promotion(0)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/gemm_sweep.json", "w"), indent=1)
