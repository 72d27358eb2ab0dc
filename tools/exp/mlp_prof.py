"""Kernel-level profile of one small-MLP training step replayed as a CUDA graph."""
import os, sys, json
from collections import defaultdict
sys.path.insert(0, os.getcwd())
import torch
from torch.profiler import profile, ProfilerActivity
import paper_2011_11188_b200 as s3
from paper_2011_11188_b200.mlp import DenseNet
h = s3.Handle(0)
sizes, B = ([4096, 4096, 4096, 4096, 1024], 4096) if os.environ.get("BIG") else ([1024, 1024, 1024, 10], 512)
X = torch.randn((B, sizes[0]), device="cuda")
y = torch.randint(0, sizes[-1], (B,), device="cuda", dtype=torch.int32)
net = DenseNet(sizes, seed=0, mode="three", h=h)
replay, _loss = net.capture_step(X, y, 0.01)
for _ in range(5): replay()
torch.cuda.synchronize()
reps = 50
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(reps): replay()
    torch.cuda.synchronize()
per = defaultdict(lambda: [0, 0.0])
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        k = e.name.replace("void ", "").replace("split3::(anonymous namespace)::", "")[:48]
        per[k][0] += 1; per[k][1] += e.device_time_total
tot = sum(v[1] for v in per.values())
for k, v in sorted(per.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:50s} {v[0]/reps:5.1f}/step {v[1]/reps:8.1f} us/step  {v[1]/max(v[0],1):7.2f} us each")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps): replay()
e1.record(); torch.cuda.synchronize()
print("step us", 1e3 * e0.elapsed_time(e1) / reps, "sum kernel us", tot / reps)
