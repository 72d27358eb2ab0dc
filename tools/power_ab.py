"""Sustained A/B of experimental builds under the power cap (one GPU): each library runs the
N = 16384 call back to back for --secs seconds in its own process; rounds alternate the libraries
so clock drift hits all of them.  Reports GEMM-kernel FP16 TFLOP/s, median SM clock and power.

  python tools/power_ab.py --tags base,hint,sleep --rounds 3 --secs 4
  python tools/power_ab.py --tags base,base@PAB_PROMO=4       (tag@ENV=VAL: same library, child env)
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if os.environ.get("PAB_CHILD"):
    if os.environ.get("EXP_ROOT"):   # another checkout's package (tools/exp/<tag>/, git-ignored)
        sys.path.insert(0, os.environ["EXP_ROOT"])
    import pynvml
    import torch

    import paper_2011_11188_b200 as s3
    if os.environ.get("EXP_LIB"):   # experimental build of the same sources (A/B runs only)
        s3.split3.LIB_PATH = os.environ["EXP_LIB"]
    from workloads import torch_matrix

    n, secs = int(os.environ["PAB_N"]), float(os.environ["PAB_SECS"])
    terms = int(os.environ.get("PAB_TERMS", "3"))   # 3 or 4 (four_term)
    pynvml.nvmlInit()
    nv = pynvml.nvmlDeviceGetHandleByIndex(0)
    h = s3.Handle(0)
    if os.environ.get("PAB_PROMO"):
        h.set_promotion(int(os.environ["PAB_PROMO"]))
    if os.environ.get("PAB_WAVE") == "0":
        h.set_wave_sync(False)
    A = torch_matrix("uniform", n, n, seed=0)
    B = torch_matrix("uniform", n, n, seed=1)
    C = torch.empty((n, n), device="cuda")
    for _ in range(3):
        h.sgemm(A, B, out=C, four_term=terms == 4)
    torch.cuda.synchronize()
    clk, pw, stop = [], [], [False]

    def poll():
        while not stop[0]:
            clk.append(pynvml.nvmlDeviceGetClockInfo(nv, pynvml.NVML_CLOCK_SM))
            pw.append(pynvml.nvmlDeviceGetPowerUsage(nv) / 1e3)
            time.sleep(0.02)
    th = threading.Thread(target=poll)
    th.start()
    h.timing_enable(True)
    h.timing_read()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0, k = time.time(), 0
    while time.time() - t0 < secs:
        h.sgemm(A, B, out=C, four_term=terms == 4)
        k += 1
        if k % 8 == 0:
            torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    stop[0] = True
    th.join()
    _, gm, nc = h.timing_read()
    clk.sort()
    pw.sort()
    print(json.dumps({"gemm_tflops": 2.0 * terms * n ** 3 / (gm / nc / 1e3) / 1e12,
                      "call_tflops": 2.0 * n ** 3 * k / (e0.elapsed_time(e1) / 1e3) / 1e12,
                      "sm_mhz": clk[len(clk) // 2], "power_w": pw[len(pw) // 2], "calls": k}))
    sys.exit(0)

p = argparse.ArgumentParser()
p.add_argument("--tags", default="base")
p.add_argument("--rounds", type=int, default=3)
p.add_argument("--secs", type=float, default=4.0)
p.add_argument("--n", type=int, default=16384)
a = p.parse_args()
res = {t: [] for t in a.tags.split(",")}
for r in range(a.rounds):
    for tag in res:
        env = dict(os.environ, PAB_CHILD="1", PAB_N=str(a.n), PAB_SECS=str(a.secs))
        lib, *kv = tag.split("@")
        for item in kv:
            k, v = item.split("=")
            env[k] = v
        if lib != "base" and os.path.isdir(os.path.join(ROOT, "tools", "exp", lib)):
            env["EXP_ROOT"] = os.path.join(ROOT, "tools", "exp", lib)
        elif lib != "base":
            env["EXP_LIB"] = os.path.join(ROOT, "tools", "exp", f"libsplit3_{lib}.so")
        out = subprocess.run([sys.executable, __file__], env=env, capture_output=True, text=True)
        try:
            res[tag].append(json.loads(out.stdout.strip().splitlines()[-1]))
        except Exception:
            res[tag].append({"error": out.stderr[-400:]})
        print(tag, res[tag][-1], flush=True)
summary = {}
for tag, rs in res.items():
    ok = [x for x in rs if "gemm_tflops" in x]
    if ok:
        summary[tag] = {k: sorted(x[k] for x in ok)[len(ok) // 2] for k in ("gemm_tflops", "call_tflops", "sm_mhz", "power_w")}
        summary[tag]["tflops_per_ghz"] = summary[tag]["gemm_tflops"] / (summary[tag]["sm_mhz"] / 1e3)
print(json.dumps(summary))
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump({"runs": res, "median": summary}, open(os.path.join(ROOT, "gpurun_out", "power_ab.json"), "w"), indent=1)
