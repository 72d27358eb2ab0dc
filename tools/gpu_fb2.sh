# fused B with direct loads: tests + GEMM-kernel rates (fused vs separate) + whole-call bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused_b.py -x -q > gpurun_out/fb2_tests.log 2>&1; echo "fused-b tests rc=$?"; tail -2 gpurun_out/fb2_tests.log
for shp in "8192 8192 8192" "256 8192 8192" "1024 8192 8192" "2048 8192 8192" "4096 8192 8192" "256 4096 4096"; do
  SPLIT3_FUSE_B=2 timeout 120 python tools/exp_ab.py time $shp base | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fused', d['M'],d['N'],d['K'], round(d['fp16_tflops'],1))"
  SPLIT3_FUSE_B=0 timeout 120 python tools/exp_ab.py time $shp base | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('separate', d['M'],d['N'],d['K'], round(d['fp16_tflops'],1))"
done
timeout 900 python tools/fused_b_bench.py --reps 20 > gpurun_out/fb2_bench.log 2>&1; echo "fb bench rc=$?"; python - <<'PY'
import json
for ln in open("gpurun_out/fb2_bench.log"):
    if ln.startswith("{"):
        d = json.loads(ln); print(d["M"], d["N"], d["K"], "sep", round(d["ms_separate"], 4), "fused", round(d["ms_fused"], 4), "presplit", round(d["ms_presplit_b"], 4))
PY
timeout 900 python tools/fused_b_bench.py --reps 20 --transb --shapes 256x8192x8192,1024x8192x8192,4096x8192x8192 > gpurun_out/fb2_bench_t.log 2>&1; echo "fb bench transB rc=$?"; python - <<'PY'
import json
for ln in open("gpurun_out/fb2_bench_t.log"):
    if ln.startswith("{"):
        d = json.loads(ln); print("transB", d["M"], d["N"], d["K"], "sep", round(d["ms_separate"], 4), "fused", round(d["ms_fused"], 4))
PY
