# N > 1 flow rehearsal on one GPU (gloo, every rank on cuda:0; not a measurement), the NCCL group
# test, and the reference arm under torchrun (rank 0 prints, the others exit 0)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dist_single.py -q -x > gpurun_out/rd_tests.log 2>&1; echo "dist single rc=$?"; tail -1 gpurun_out/rd_tests.log
for n in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29$((500+n)) \
  bench.py --gpus $n --steps 3 --warmup 3 --dist-backend gloo --global-n 8192 --e2e-steps 2 --sustained-s 0 > gpurun_out/rd_bench_$n.log 2>&1
echo "rehearsal N=$n rc=$? lines=$(grep -c '^{' gpurun_out/rd_bench_$n.log)"; grep '^{' gpurun_out/rd_bench_$n.log | cut -c1-400
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29510 \
  bench.py --impl reference --gpus 2 --steps 3 --warmup 1 > gpurun_out/rd_ref2.log 2>&1
echo "ref N=2 rc=$? lines=$(grep -c '^{' gpurun_out/rd_ref2.log)"; grep '^{' gpurun_out/rd_ref2.log | cut -c1-500
