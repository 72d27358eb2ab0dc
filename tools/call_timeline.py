"""CUPTI timeline (torch.profiler) of split3_sgemm calls at N (default 16384): kernel intervals and
the gaps between them (the split phase's share of the step).  Writes gpurun_out/call_timeline.json."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2011_11188_b200 as s3  # noqa: E402
from workloads import torch_matrix  # noqa: E402

n = int(os.environ.get("CT_N", "16384"))
A = torch_matrix("uniform", n, n, seed=0)
B = torch_matrix("uniform", n, n, seed=1)
C = torch.empty((n, n), device="cuda")
h = s3.Handle(0)
for _ in range(3):
    h.sgemm(A, B, out=C)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        h.sgemm(A, B, out=C)
    torch.cuda.synchronize()
evs = sorted((e for e in prof.events() if e.device_type.name == "CUDA"), key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
rows = [((e.time_range.start - t0) / 1e3, (e.time_range.end - t0) / 1e3, e.name) for e in evs]
for s0, e0, nm in rows:
    print(f"{s0:10.4f} {e0:10.4f} {e0 - s0:9.4f}  {nm[:60]}")
gaps = [rows[i + 1][0] - rows[i][1] for i in range(len(rows) - 1)]
print("gaps_ms", [round(g, 4) for g in gaps])
json.dump({"n": n, "timeline_ms": [[round(a, 4), round(b, 4), c] for a, b, c in rows], "gaps_ms": gaps},
          open("gpurun_out/call_timeline.json", "w"), indent=1)
