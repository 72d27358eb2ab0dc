# stream-K: tests, D3 config table, fused-B bench, full GPU suite
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_streamk.py -q -x > gpurun_out/sk_tests.log 2>&1; echo "streamk tests rc=$?"; tail -3 gpurun_out/sk_tests.log
timeout 900 python tools/config_table.py > gpurun_out/sk_config.log 2>&1; echo "config table rc=$?"; grep -E "D3|D2 N=4096" gpurun_out/sk_config.log | head -24
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/sk_all.log 2>&1; echo "all gpu tests rc=$?"; tail -3 gpurun_out/sk_all.log
