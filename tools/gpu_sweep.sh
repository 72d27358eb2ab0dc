mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv -lms 500 > gpurun_out/sweep_clocks.csv &
SMI=$!
timeout 600 python tools/gemm_sweep.py ${SWEEP_ARGS} 2>&1 | tail -40
kill $SMI
