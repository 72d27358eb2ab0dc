# Round-2 first GPU pass: smoke, whole -m gpu suite, one bench line.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r02a_smi.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/r02a_smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r02a_gpu_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r02a_gpu_tests.log
timeout 900 python bench.py > gpurun_out/r02a_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r02a_bench.log
