"""Timeline (CUPTI via torch.profiler) of one split3_sgemm_host call at N = 16384: start/end of
every memcpy and kernel relative to the first activity.  Prints a compact table."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2011_11188_b200 as s3  # noqa: E402
from workloads import torch_matrix  # noqa: E402

n = int(os.environ.get("E2E_N", "16384"))
h = s3.Handle(0)
A = torch_matrix("uniform", n, n, seed=0)
B = torch_matrix("uniform", n, n, seed=1)
Ah = torch.empty((n, n), dtype=torch.float32, pin_memory=True); Ah.copy_(A)
Bh = torch.empty((n, n), dtype=torch.float32, pin_memory=True); Bh.copy_(B)
Ch = torch.empty((n, n), dtype=torch.float32, pin_memory=True)
del A, B
torch.cuda.empty_cache()
for _ in range(2):
    h.sgemm_host_ptr(n, n, n, Ah.data_ptr(), Bh.data_ptr(), Ch.data_ptr(), 0)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    h.sgemm_host_ptr(n, n, n, Ah.data_ptr(), Bh.data_ptr(), Ch.data_ptr(), 0)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
t0 = min(e.time_range.start for e in evs)
rows = sorted(((e.time_range.start - t0) / 1e3, (e.time_range.end - t0) / 1e3, e.name[:40]) for e in evs)
for s, e, nm in rows:
    print(f"{s:8.2f} {e:8.2f} {e - s:7.2f}  {nm}")
