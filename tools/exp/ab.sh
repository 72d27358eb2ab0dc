python tools/call_breakdown.py 4096 16384 2>&1 | grep "{" | sed 's/^/fused /'
SPLIT3_FUSED_SCALE=0 python tools/call_breakdown.py 4096 16384 2>&1 | grep "{" | sed 's/^/twopass /'
