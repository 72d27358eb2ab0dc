python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for r in 1 2; do
python tools/call_breakdown.py 256x8192x8192 1024x8192x8192 4096 8192 16384 2>&1 | grep "{" | sed 's/^/mn /'
SPLIT3_B_MN=0 python tools/call_breakdown.py 256x8192x8192 1024x8192x8192 4096 8192 16384 2>&1 | grep "{" | sed 's/^/kmaj /'
done
for r in 1 2; do
EXP_REPS=30 python tools/exp_ab.py time 16384 16384 16384 base | sed 's/"base"/"mn"/'
SPLIT3_B_MN=0 EXP_REPS=30 python tools/exp_ab.py time 16384 16384 16384 base | sed 's/"base"/"kmaj"/'
done
