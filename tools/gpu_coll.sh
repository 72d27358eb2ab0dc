# collector-reuse A/B: bitwise vs the previous build, GEMM parity subset, sustained power A/B, fused-B GEMM times
mkdir -p gpurun_out
timeout 600 python - > gpurun_out/coll_bitwise.log 2>&1 <<'PY'
import subprocess, sys, os, json
code = r'''
import os, sys, torch, hashlib
sys.path.insert(0, ".")
import paper_2011_11188_b200 as s3
if os.environ.get("EXP_LIB"): s3.split3.LIB_PATH = os.environ["EXP_LIB"]
from workloads import torch_matrix
h = s3.Handle(0)
out = {}
for (M, N, K, kind) in [(4096, 4096, 4096, "uniform"), (16384, 16384, 4096, "loguni"), (256, 8192, 8192, "glorot"), (2304, 1152, 777, "uniform")]:
    A = torch_matrix(kind, M, K, seed=1); B = torch_matrix(kind, K, N, seed=2)
    for terms in (3, 4, 1):
        C = h.sgemm(A, B, four_term=terms == 4, one_term=terms == 1)
        torch.cuda.synchronize()
        out[f"{M}x{N}x{K}/{kind}/{terms}"] = hashlib.sha256(C.cpu().numpy().tobytes()).hexdigest()
print(repr(out))
'''
res = {}
for lib in ("paper_2011_11188_b200/libsplit3.so", "tools/exp/libsplit3_nocoll.so"):
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, EXP_LIB=lib), capture_output=True, text=True)
    res[lib] = eval(r.stdout.strip().splitlines()[-1])
a, b = res.values()
print("bitwise equal:", a == b, {k: a[k] == b[k] for k in a})
PY
echo "bitwise rc=$?"; cat gpurun_out/coll_bitwise.log | tail -2
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused_b.py -q -x > gpurun_out/coll_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/coll_tests.log
timeout 1500 python tools/power_ab.py --tags nocoll,coll --rounds 4 --secs 4 > gpurun_out/coll_power.log 2>&1; echo "power rc=$?"; tail -1 gpurun_out/coll_power.log
for shp in "8192 8192 8192" "256 8192 8192" "1024 8192 8192"; do
  for t in nocoll coll; do SPLIT3_FUSE_B=2 timeout 120 python tools/exp_ab.py time $shp $t | cut -c 1-220; done
  SPLIT3_FUSE_B=0 timeout 120 python tools/exp_ab.py time $shp coll | cut -c 1-220
done
