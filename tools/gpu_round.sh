# One measured round: plain bench (JSON line), ncu launch list of the same bench command,
# one ncu --set full capture of the GEMM kernel.  Outputs under gpurun_out/.
mkdir -p gpurun_out
TAG=${TAG:-r01}
BARGS=${BARGS:-"--steps 30 --warmup 5"}
timeout 900 python bench.py $BARGS > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_$TAG.log
LARGS="--steps 3 --warmup 3 --no-e2e --no-cpu --sustained-s 0"
timeout 600 python bench.py $LARGS > gpurun_out/bench_launch_plain_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py $LARGS > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm3 -s 3 -c 1 \
    -o gpurun_out/gemm3_full_$TAG python bench.py $LARGS > gpurun_out/ncu_full_$TAG.log 2>&1
echo "full rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:"split" -s 6 -c 2 \
    -o gpurun_out/split_t_full_$TAG python bench.py $LARGS > gpurun_out/ncu_split_$TAG.log 2>&1
echo "split full rc=$?"
timeout 600 python tools/run_sgemm.py --n 8192 --reps 2 --terms 6 > gpurun_out/bf16_plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:gemm3 -s 1 -c 1 \
    -o gpurun_out/gemm3_bf16x3_full_$TAG python tools/run_sgemm.py --n 8192 --reps 2 --terms 6 > gpurun_out/ncu_bf16_$TAG.log 2>&1
echo "bf16x3 full rc=$?"
