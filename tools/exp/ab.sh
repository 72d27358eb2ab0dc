for r in 1 2; do
python tools/split_bench.py 16384 | sed 's/^/base /'
SPLIT3_EXPERIMENT_LIB=tools/exp/libsplit3_rot.so python tools/split_bench.py 16384 | sed 's/^/rot /'
python tools/split_bench.py 4096 | sed 's/^/base /'
SPLIT3_EXPERIMENT_LIB=tools/exp/libsplit3_rot.so python tools/split_bench.py 4096 | sed 's/^/rot /'
done
SPLIT3_EXPERIMENT_LIB=tools/exp/libsplit3_rot.so python -m pytest tests -x -q -m gpu -k "plane or split or transpose or presplit" 2>&1 | tail -2
