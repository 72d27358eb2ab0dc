# fused-B (NEXT #2) experiment: GEMM-kernel time, separate split (FUSE_B=0) vs fused (=2)
mkdir -p gpurun_out
for i in 1 2 3; do timeout 200 python -m pytest tests/test_gpu_fused_b.py -x -q 2>&1 | tail -1; done
for shp in "8192 8192 8192" "256 8192 8192" "1024 8192 8192" "256 4096 4096"; do
  SPLIT3_FUSE_B=0 timeout 120 python tools/exp_ab.py time $shp base | cut -c 80-200
  SPLIT3_FUSE_B=2 timeout 120 python tools/exp_ab.py time $shp base $EXP_TAGS | cut -c 80-200
done
