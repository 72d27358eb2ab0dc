# Round-2 pass d: overlap timeline (fixed ordering), full GPU suite on the cleaned kernel source, bench
mkdir -p gpurun_out
timeout 600 python tools/overlap_timeline.py > gpurun_out/r02d_overlap.log 2>&1; echo "overlap rc=$?"
grep -E "^\{|^---" gpurun_out/r02d_overlap.log
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r02d_gpu_tests.log 2>&1; echo "all tests rc=$?"
tail -3 gpurun_out/r02d_gpu_tests.log
timeout 900 python bench.py > gpurun_out/r02d_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r02d_bench.log | cut -c1-600
