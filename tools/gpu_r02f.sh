mkdir -p gpurun_out
TAG=${TAG:-r02f}
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputests_$TAG.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/gputests_$TAG.log | grep -E 'passed|failed|FAILED|Error' | head -20
timeout 900 python tools/power_ab.py --tags base,old --rounds 4 --secs 4 > gpurun_out/power_ab_$TAG.log 2>&1; echo "power ab rc=$?"
tail -1 gpurun_out/power_ab_$TAG.log
cp gpurun_out/power_ab.json gpurun_out/power_ab_$TAG.json
