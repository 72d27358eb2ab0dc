"""cuBLAS fp16 GEMM (fp32 accumulate) sustained on the split's own planes (A1 x B1, A2 x B1):
separates data-dependent power from kernel efficiency when comparing with gemm3."""
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

pynvml.nvmlInit()
nv = pynvml.nvmlDeviceGetHandleByIndex(0)
n = 16384
h = s3.Handle(0)
A = torch_matrix("uniform", n, n, seed=0)
B = torch_matrix("uniform", n, n, seed=1)
d = torch.zeros(2, device="cuda")
h.maxabs(A, d[0:1]); h.maxabs(B, d[1:2])
A1, A2, _ = h.split(A, d[0:1])
B1, B2, _ = h.split(B, d[1:2], transpose=True)
del A, B
a1, a2 = A1[:, :n].view(torch.float16), A2[:, :n].view(torch.float16)
b1 = B1[:, :n].view(torch.float16).t()
torch.backends.cuda.matmul.allow_fp16_reduced_precision_reduction = False
res = []
for name, (x, y) in {"cuBLAS fp16 A1 x B1 (split planes)": (a1, b1), "cuBLAS fp16 A2 x B1 (split planes)": (a2, b1),
                     "cuBLAS fp16 rand[0,1)": (torch.rand((n, n), device="cuda").half(),
                                               torch.rand((n, n), device="cuda").half())}.items():
    C = torch.matmul(x, y)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); torch.matmul(x, y, out=C); torch.cuda.synchronize()
    reps = max(3, int(4.0 / (time.perf_counter() - t0)))
    clk, stop = [], [False]

    def samp():
        while not stop[0]:
            clk.append(pynvml.nvmlDeviceGetClockInfo(nv, pynvml.NVML_CLOCK_SM)); time.sleep(0.01)

    th = threading.Thread(target=samp, daemon=True); th.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        torch.matmul(x, y, out=C)
    e1.record(); torch.cuda.synchronize(); stop[0] = True; th.join()
    ms = e0.elapsed_time(e1) / reps
    r = {"impl": name, "tflops": 2.0 * n ** 3 / (ms / 1e3) / 1e12, "sm_mhz": sorted(clk)[len(clk) // 2]}
    print(json.dumps(r), flush=True)
    res.append(r)
json.dump(res, open("gpurun_out/cublas_on_planes.json", "w"), indent=1)
