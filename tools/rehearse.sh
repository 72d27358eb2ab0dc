# round-end rehearsal: clean build, smoke, default bench, reference arm (one GPU)
mkdir -p gpurun_out
rm -f paper_2011_11188_b200/*.so oracle/*.so
timeout 600 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/rh_build.log 2>&1; echo "build rc=$?"
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rh_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/rh_smoke.log
timeout 900 python bench.py > gpurun_out/rh_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/rh_bench.log
timeout 900 python bench.py --impl reference > gpurun_out/rh_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/rh_ref.log
