python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for r in 1 2; do
python tools/call_breakdown.py 1024 2048 4096 8192 2>&1 | grep "{" | sed 's/^/pdl /'
SPLIT3_EXPERIMENT_LIB=tools/exp/libsplit3_nopdl.so python tools/call_breakdown.py 1024 2048 4096 8192 2>&1 | grep "{" | sed 's/^/nopdl /'
done
