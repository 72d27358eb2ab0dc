# Round-2 pass: binding + dist tests, then the whole -m gpu suite
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_binding.py tests/test_gpu_dist_single.py tests/test_gpu_dist_gloo_cuda.py -q -x > gpurun_out/r02b_dist.log 2>&1; echo "dist tests rc=$?"
tail -30 gpurun_out/r02b_dist.log
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r02b_gpu_tests.log 2>&1; echo "all tests rc=$?"
tail -30 gpurun_out/r02b_gpu_tests.log
