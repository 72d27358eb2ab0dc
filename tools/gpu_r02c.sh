# Round-2 pass c: new parity tests, overlap timeline, bench N=1, 1-GPU D5 path, split-kernel ncu
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "vs_oracle or distributions or full_4096" -s > gpurun_out/r02c_parity.log 2>&1; echo "parity rc=$?"
grep -E "passed|failed|max_err" gpurun_out/r02c_parity.log | tail -5
timeout 600 python tools/overlap_timeline.py > gpurun_out/r02c_overlap.log 2>&1; echo "overlap rc=$?"
grep -E "^\{|^---" gpurun_out/r02c_overlap.log
timeout 900 python bench.py > gpurun_out/r02c_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r02c_bench.log
timeout 900 python bench.py --global-n 32768 --steps 3 --warmup 3 --no-cpu --sustained-s 0 --e2e-steps 2 > gpurun_out/r02c_d5_1gpu.log 2>&1; echo "dist-path bench rc=$?"
tail -1 gpurun_out/r02c_d5_1gpu.log
LARGS="--steps 3 --warmup 3 --no-e2e --no-cpu --sustained-s 0"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  -k regex:"maxabs|split" --log-file gpurun_out/r02c_split_ncu.csv python bench.py $LARGS > gpurun_out/r02c_split_ncu.log 2>&1; echo "split ncu rc=$?"
