mkdir -p gpurun_out
TAG=${TAG:-r02k}
timeout 1500 python -m pytest -q -p no:cacheprovider tests/test_gpu_fold.py > gpurun_out/fold_tests_$TAG.log 2>&1; rc=$?; echo "fold tests rc=$rc"
grep -E 'passed|failed|^FAILED' gpurun_out/fold_tests_$TAG.log | head -20
timeout 1200 python tools/power_ab.py --tags base,base@SPLIT3_FOLD=1 --rounds 4 --secs 4 > gpurun_out/fold_ab_$TAG.log 2>&1; echo "fold ab rc=$?"
tail -1 gpurun_out/fold_ab_$TAG.log
cp gpurun_out/power_ab.json gpurun_out/fold_ab_$TAG.json
timeout 1200 python tools/power_ab.py --tags base@PAB_TERMS=4,base@SPLIT3_FOLD=1@PAB_TERMS=4 --rounds 3 --secs 4 > gpurun_out/fold4_ab_$TAG.log 2>&1; echo "fold4 ab rc=$?"
tail -1 gpurun_out/fold4_ab_$TAG.log
cp gpurun_out/power_ab.json gpurun_out/fold4_ab_$TAG.json
