# Final measured round: bench + ncu (tools/gpu_round.sh), the per-config table, a 4-term (folded)
# GEMM capture.  Outputs under gpurun_out/.
mkdir -p gpurun_out
TAG=${TAG:-r02m}
TAG=$TAG bash tools/gpu_round.sh
timeout 600 python tools/run_sgemm.py --n 8192 --reps 2 --terms 4 > gpurun_out/fold4_plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm3 -s 1 -c 1 \
    -o gpurun_out/gemm3_fold4_full_$TAG python tools/run_sgemm.py --n 8192 --reps 2 --terms 4 > gpurun_out/ncu_fold4_$TAG.log 2>&1
echo "fold4 full rc=$?"
timeout 1500 python tools/config_table.py > gpurun_out/cfg_$TAG.log 2>&1; echo "cfg rc=$?"
cp gpurun_out/config_table.json gpurun_out/config_table_$TAG.json
