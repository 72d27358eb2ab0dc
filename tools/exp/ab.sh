for r in 1 2; do
python tools/call_breakdown.py 64 256x1024x1024 256x4096x4096 256x8192x8192 1024 1024x4096x4096 4096 2>&1 | grep "{" | sed 's/^/new /'
SPLIT3_EXPERIMENT_LIB=tools/exp/libsplit3_prev.so python tools/call_breakdown.py 64 256x1024x1024 256x4096x4096 256x8192x8192 1024 1024x4096x4096 4096 2>&1 | grep "{" | sed 's/^/prev /'
SPLIT3_EXPERIMENT_LIB=tools/exp/libsplit3_nosplit.so python tools/call_breakdown.py 64 256x1024x1024 256x4096x4096 256x8192x8192 1024 1024x4096x4096 4096 2>&1 | grep "{" | sed 's/^/nosplit /'
done
