mkdir -p gpurun_out
TAG=${TAG:-r02n}
timeout 300 python tools/host_overhead.py 64 256 1024 > gpurun_out/host_ovh_fused_$TAG.log 2>&1; echo "rc=$?"
SPLIT3_FUSE_B=0 timeout 300 python tools/host_overhead.py 64 256 1024 > gpurun_out/host_ovh_prep_$TAG.log 2>&1; echo "rc=$?"
cat gpurun_out/host_ovh_fused_$TAG.log gpurun_out/host_ovh_prep_$TAG.log
timeout 300 python tools/config_table.py --only "D1" > gpurun_out/cfg_d1_$TAG.log 2>&1; python -c "import json; print(json.load(open('gpurun_out/config_table.json')))"
SPLIT3_FUSE_B=0 timeout 300 python tools/config_table.py --only "D1" > gpurun_out/cfg_d1b_$TAG.log 2>&1; python -c "import json; print(json.load(open('gpurun_out/config_table.json')))"
