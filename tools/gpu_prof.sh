mkdir -p gpurun_out
N=${PROF_N:-8192}
python tools/run_sgemm.py --n $N --reps 2 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/run_sgemm.py --n $N --reps 2 > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${PROF_K:-gemm3} -s 1 -c 1 -o gpurun_out/prof_${PROF_TAG:-gemm} python tools/run_sgemm.py --n $N --reps 2 > gpurun_out/ncu_full.log 2>&1
echo "rc=$?"
tail -3 gpurun_out/ncu_full.log
