mkdir -p gpurun_out
python tools/run_sgemm.py --n ${PROF_N:-16384} --k ${PROF_K:-4096} --reps 2 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm3 -s 1 -c 1 -o gpurun_out/prof_${PROF_TAG:-k4096} python tools/run_sgemm.py --n ${PROF_N:-16384} --k ${PROF_K:-4096} --reps 2 > gpurun_out/ncu_full2.log 2>&1
echo "rc=$?"
