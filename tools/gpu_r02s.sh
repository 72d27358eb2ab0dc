mkdir -p gpurun_out
TAG=${TAG:-r02s}
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gputests_$TAG.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/gputests_$TAG.log
for n in 16384 4096; do
  timeout 900 python tools/power_ab.py --n $n --tags base,old --rounds 4 --secs 3 > gpurun_out/split2_ab_${n}_$TAG.log 2>&1; echo "ab $n rc=$?"
  tail -1 gpurun_out/split2_ab_${n}_$TAG.log
  cp gpurun_out/power_ab.json gpurun_out/split2_ab_${n}_$TAG.json
done
timeout 600 python tools/call_timeline.py > gpurun_out/call_timeline_$TAG.log 2>&1; grep gaps gpurun_out/call_timeline_$TAG.log; head -4 gpurun_out/call_timeline_$TAG.log | cut -c1-100
