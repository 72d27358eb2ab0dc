python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for r in 1 2; do
python tools/call_breakdown.py 64 256x1024x1024 512x1024x1024 1024 2048 256x4096x4096 2>&1 | grep "{" | sed 's/^/prep /'
SPLIT3_PREP_MAX=0 python tools/call_breakdown.py 64 256x1024x1024 512x1024x1024 1024 2048 256x4096x4096 2>&1 | grep "{" | sed 's/^/noprep /'
done
