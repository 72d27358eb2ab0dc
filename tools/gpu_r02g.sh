mkdir -p gpurun_out
TAG=${TAG:-r02g}
timeout 1800 python -m pytest -q -p no:cacheprovider tests/test_gpu_fused_a.py tests/test_gpu_mn_major.py tests/test_gpu_prep.py \
   tests/test_gpu_stored_planes.py "tests/test_gpu_parity.py::test_host_pipeline_bitwise_equals_device" tests/test_gpu_fused_b.py \
   > gpurun_out/tests_$TAG.log 2>&1; echo "tests rc=$?"
grep -E 'passed|failed|^FAILED' gpurun_out/tests_$TAG.log | head -20
timeout 600 python tools/small_fused_bench.py > gpurun_out/small_fused_$TAG.log 2>&1; echo "small rc=$?"
