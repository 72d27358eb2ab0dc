"""Training-step throughput of a wide dense network whose GEMMs run as split-3 (NEXT #3).

Effective TFLOP/s counts the 3 GEMMs per layer (forward, dW, dX; 6*B*in*out FLOPs). Context: the
same step in plain torch fp32 (cuBLAS SGEMM, TF32 off) on the same box.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2011_11188_b200 as s3  # noqa: E402
from paper_2011_11188_b200.mlp import DenseNet  # noqa: E402

h = s3.Handle(0)
res = []


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def run(sizes, B, torch_ref=True):
    X = torch.randn((B, sizes[0]), device="cuda")
    y = torch.randint(0, sizes[-1], (B,), device="cuda", dtype=torch.int32)
    flops = sum(6.0 * B * a * b for a, b in zip(sizes[:-1], sizes[1:]))
    tag = f"{'x'.join(map(str, sizes))} batch {B}"
    for mode in ("three", "one", "four"):
        net = DenseNet(sizes, seed=0, mode=mode, h=h)
        ms = timeit(lambda: net.step_device(X, y, 1e-3))
        res.append({"net": tag, "impl": f"split3 {mode}-term", "ms_per_step": ms,
                    "eff_tflops": flops / (ms / 1e3) / 1e12})
        print(json.dumps(res[-1]), flush=True)
        if mode == "three":
            replay, _ = net.capture_step(X, y, 1e-3)
            ms = timeit(replay)
            res.append({"net": tag, "impl": "split3 three-term, CUDA graph", "ms_per_step": ms,
                        "eff_tflops": flops / (ms / 1e3) / 1e12})
            print(json.dumps(res[-1]), flush=True)
    if not torch_ref:
        return
    torch.backends.cuda.matmul.allow_tf32 = False
    Ws = [torch.randn((a, b), device="cuda") * (2.0 / (a + b)) ** 0.5 for a, b in zip(sizes[:-1], sizes[1:])]
    bs = [torch.zeros(b, device="cuda") for b in sizes[1:]]
    for t in Ws + bs:
        t.requires_grad_(True)
    yl = y.long()

    def torch_step():
        hcur = X
        for i, (w, b) in enumerate(zip(Ws, bs)):
            hcur = hcur @ w + b
            if i < len(Ws) - 1:
                hcur = torch.relu(hcur)
        loss = torch.nn.functional.cross_entropy(hcur, yl)
        gs = torch.autograd.grad(loss, Ws + bs)
        with torch.no_grad():
            for p, g in zip(Ws + bs, gs):
                p -= 1e-3 * g

    ms = timeit(torch_step, reps=5)
    res.append({"net": tag, "impl": "torch fp32 (cuBLAS SGEMM, TF32 off)", "ms_per_step": ms,
                "eff_tflops": flops / (ms / 1e3) / 1e12})
    print(json.dumps(res[-1]), flush=True)


run([4096, 4096, 4096, 4096, 1024], 4096)
run([1024, 1024, 1024, 10], 512)
os.makedirs("gpurun_out", exist_ok=True)
json.dump({"results": res}, open("gpurun_out/mlp_bench.json", "w"), indent=1)
