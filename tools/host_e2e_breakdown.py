"""e2e (host-buffer) call at N = 16384 vs the PCIe bounds (one GPU).

PCIe: pinned H2D / D2H alone and both directions at once; the host call for several row-block
counts (SPLIT3_HOST_BLOCKS; 0 = automatic).  Writes gpurun_out/host_e2e.json.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
n = int(os.environ.get("E2E_N", "16384"))

if os.environ.get("E2E_CHILD"):
    import torch

    import paper_2011_11188_b200 as s3
    from workloads import torch_matrix

    h = s3.Handle(0)
    A = torch_matrix("uniform", n, n, seed=0)
    B = torch_matrix("uniform", n, n, seed=1)
    Ah = torch.empty((n, n), dtype=torch.float32, pin_memory=True); Ah.copy_(A)
    Bh = torch.empty((n, n), dtype=torch.float32, pin_memory=True); Bh.copy_(B)
    Ch = torch.empty((n, n), dtype=torch.float32, pin_memory=True)
    del A, B
    torch.cuda.empty_cache()
    h.sgemm_host_ptr(n, n, n, Ah.data_ptr(), Bh.data_ptr(), Ch.data_ptr(), 0)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        h.sgemm_host_ptr(n, n, n, Ah.data_ptr(), Bh.data_ptr(), Ch.data_ptr(), 0)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(json.dumps({"blocks": os.environ.get("SPLIT3_HOST_BLOCKS", "0"),
                      "panels": os.environ.get("SPLIT3_HOST_PANELS", "0"), "ms": ts[len(ts) // 2],
                      "launches": h.last_launch_count(), "redo": h.host_redo_count()}))
    sys.exit(0)

import torch  # noqa: E402

res = {"n": n}
m = 256 * 2 ** 20
hb = torch.empty(2 * m, dtype=torch.float32, pin_memory=True)
hc = torch.empty(m, dtype=torch.float32, pin_memory=True)
db = torch.empty(2 * m, dtype=torch.float32, device="cuda")
dc = torch.empty(m, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def ev_time(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


res["h2d_2GiB_ms"] = ev_time(lambda: db.copy_(hb, non_blocking=True))
res["d2h_1GiB_ms"] = ev_time(lambda: hc.copy_(dc, non_blocking=True))


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        db.copy_(hb, non_blocking=True)
    with torch.cuda.stream(s2):
        hc.copy_(dc, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)


res["h2d_2GiB_with_d2h_1GiB_ms"] = ev_time(both)
del hb, hc, db, dc
torch.cuda.empty_cache()
runs = []
for blocks, panels in (("0", "0"), ("0", "1"), ("0", "2"), ("0", "4"), ("1", "0"), ("4", "0"), ("8", "0")):
    env = dict(os.environ, E2E_CHILD="1", SPLIT3_HOST_BLOCKS=blocks, SPLIT3_HOST_PANELS=panels)
    out = subprocess.run([sys.executable, __file__], env=env, capture_output=True, text=True)
    try:
        runs.append(json.loads(out.stdout.strip().splitlines()[-1]))
    except Exception:
        runs.append({"blocks": blocks, "error": out.stderr[-500:]})
res["host_call"] = runs
print(json.dumps(res))
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(res, open(os.path.join(ROOT, "gpurun_out", "host_e2e.json"), "w"), indent=1)
