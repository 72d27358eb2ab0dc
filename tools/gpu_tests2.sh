mkdir -p gpurun_out
free -g | head -2
timeout 1800 python -m pytest ${TEST_FILES:-tests/test_gpu_configs.py} -q -x -s > gpurun_out/gpu_tests2.log 2>&1; echo "tests rc=$?"
grep -E "passed|failed|Error|error" gpurun_out/gpu_tests2.log | tail -5
grep "config" gpurun_out/gpu_tests2.log | tail -20
