"""A/B timing of experimental builds (extra -D flags, e.g. SPLIT3_PDL=0, of the same sources; or
patched builds from tools/exp_patch_build.py).  Round 1's in-kernel cycle-counter trace build
(profiles/gemm3_trace_r01.md) was removed from the product sources in round 2.

  python tools/exp_ab.py build TAG DEFINE...     (here: nvcc -> tools/exp/libsplit3_TAG.so)
  python tools/exp_ab.py time  M N K [TAG...]    (on the GPU: GEMM-kernel time per library)
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if sys.argv[1] == "build":
    from paper_2011_11188_b200 import _build

    tag = sys.argv[2]
    out = os.path.join(ROOT, "tools", "exp", f"libsplit3_{tag}.so")
    print(_build.build(force=True, out=out, defines=sys.argv[3:]))
    sys.exit(0)

M, N, K = (int(x) for x in sys.argv[2:5])
tags = sys.argv[5:] or ["base"]
if len(tags) > 1 or os.environ.get("EXP_CHILD") is None:
    for tag in tags:
        env = dict(os.environ, EXP_CHILD="1")
        if tag != "base":
            env["EXP_LIB"] = os.path.join(ROOT, "tools", "exp", f"libsplit3_{tag}.so")
        out = subprocess.run([sys.executable, __file__, "time", str(M), str(N), str(K), tag], env=env,
                             capture_output=True, text=True)
        print(out.stdout.strip() or out.stderr[-2000:])
    sys.exit(0)

import torch  # noqa: E402

import paper_2011_11188_b200 as s3  # noqa: E402
if os.environ.get("EXP_LIB"):   # experimental build of the same sources (A/B runs only)
    s3.split3.LIB_PATH = os.environ["EXP_LIB"]
from workloads import torch_matrix  # noqa: E402

h = s3.Handle(0)
if os.environ.get("EXP_WAVE") == "0":
    h.set_wave_sync(False)
A = torch_matrix("uniform", M, K, seed=0)
B = torch_matrix("uniform", K, N, seed=1)
C = torch.empty((M, N), device="cuda")
for _ in range(3):
    h.sgemm(A, B, out=C)
torch.cuda.synchronize()
h.timing_enable(True)
h.timing_read()
reps = int(os.environ.get("EXP_REPS", "20"))
for _ in range(reps):
    h.sgemm(A, B, out=C)
torch.cuda.synchronize()
sp, gm, n = h.timing_read()
rec = {"tag": tags[0], "lib": s3.split3.LIB_PATH, "M": M, "N": N, "K": K,
       "gemm_ms": gm / n, "fp16_tflops": 3 * 2.0 * M * N * K / (gm / n / 1e3) / 1e12}
if os.environ.get("EXP_ACC"):               # accuracy of this build vs fp64 (measurement only)
    C64 = A.double() @ B.double()
    rec["e64rel"] = float((C.double() - C64).norm() / C64.norm())
    del C64
print(json.dumps(rec))
