mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -3 gpurun_out/smoke.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x ${TEST_ARGS} > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -30 gpurun_out/gpu_tests.log
cat gpurun_out/promo_sweep.json 2>/dev/null
if [ -n "$SWEEP_ARGS" ]; then timeout 600 python tools/gemm_sweep.py $SWEEP_ARGS 2>&1 | tail -20; fi
