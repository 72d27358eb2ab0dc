# Fused-A round: its GPU tests (+ the epilogue scale test, debug build, fused-B regression), the
# fused-A bench, the D3 config rows, and an ncu look at the M = 256, K = N = 8192 fused-B call.
mkdir -p gpurun_out
TAG=${TAG:-r02e}
timeout 1500 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_fused_a.py tests/test_gpu_fused_b.py \
    tests/test_gpu_debug_build.py "tests/test_gpu_parity.py::test_epilogue_scale_outside_fp32_normal_range" \
    > gpurun_out/fa_tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/fa_tests_$TAG.log
timeout 600 python tools/fused_a_bench.py > gpurun_out/fa_bench_$TAG.log 2>&1; echo "fa bench rc=$?"
timeout 600 python tools/config_table.py --only D3 > gpurun_out/cfg_d3_$TAG.log 2>&1; echo "cfg rc=$?"
cp gpurun_out/config_table.json gpurun_out/config_table_d3_$TAG.json 2>/dev/null
timeout 300 python tools/run_sgemm.py --m 256 --n 8192 --k 8192 --reps 3 > gpurun_out/m256_plain_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/m256_launches_$TAG.csv python tools/run_sgemm.py --m 256 --n 8192 --k 8192 --reps 3 \
    > gpurun_out/m256_ncu_$TAG.log 2>&1
echo "m256 launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm3 -s 2 -c 1 \
    -o gpurun_out/m256_gemm_full_$TAG python tools/run_sgemm.py --m 256 --n 8192 --k 8192 --reps 3 \
    > gpurun_out/m256_full_$TAG.log 2>&1
echo "m256 full rc=$?"
timeout 900 python tools/power_ab.py --tags base,old --rounds 4 --secs 4 > gpurun_out/power_ab_$TAG.log 2>&1; echo "power ab rc=$?"
tail -1 gpurun_out/power_ab_$TAG.log
