# fused-B GEMM (NEXT #2): one ncu --set full capture with source (stall reasons per line)
mkdir -p gpurun_out
SPLIT3_FUSE_B=2 timeout 120 python tools/exp_ab.py time ${FB_SHAPE:-8192 8192 8192} base > gpurun_out/fb_plain.log 2>&1; cat gpurun_out/fb_plain.log | cut -c1-200
SPLIT3_FUSE_B=2 EXP_REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm3 -s 3 -c 1 \
  -o gpurun_out/fb_full_${FB_TAG:-a} python tools/exp_ab.py time ${FB_SHAPE:-8192 8192 8192} base > gpurun_out/fb_ncu.log 2>&1
echo "ncu rc=$?"
