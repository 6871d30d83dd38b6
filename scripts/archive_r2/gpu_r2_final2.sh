# closing check at HEAD: full GPU suite, smoke, default bench, lap16k/c1 seam lines
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2/smoke.log 2>&1; echo "smoke rc=$?" | tee -a gpurun_out/final2/smoke.log
timeout 900 python bench.py > gpurun_out/final2/bench_c4.log 2>&1; tail -1 gpurun_out/final2/bench_c4.log | cut -c1-200
for wl in c1 lap16k; do timeout 900 python bench.py --workload $wl --no-cpu-baseline > gpurun_out/final2/bench_$wl.log 2>&1; tail -1 gpurun_out/final2/bench_$wl.log | cut -c1-160; done
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1500 -rfE > gpurun_out/final2/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final2/pytest_gpu.log
tail -6 gpurun_out/final2/pytest_gpu.log
