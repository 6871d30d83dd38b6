# closing evidence at the final HEAD: full GPU suite, smoke, default bench, C5 BASELINE shape
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/closing
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/closing/smoke.log 2>&1; echo "smoke rc=$?" | tee -a gpurun_out/closing/smoke.log
timeout 900 python bench.py > gpurun_out/closing/bench_c4.log 2>&1; tail -1 gpurun_out/closing/bench_c4.log | cut -c1-200
rm -rf /tmp/est-r3-*
EST_WORKER_LOG=1 timeout 2400 python scripts/rescale3d_bench.py > gpurun_out/closing/c5.json 2> gpurun_out/closing/c5.err; echo "c5 rc=$?"; cut -c1-700 gpurun_out/closing/c5.json
mkdir -p gpurun_out/closing/c5logs; for d in /tmp/est-r3-*; do cp -r $d/logs gpurun_out/closing/c5logs/$(basename $d) 2>/dev/null; done
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1500 -rfE > gpurun_out/closing/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/closing/pytest_gpu.log
tail -6 gpurun_out/closing/pytest_gpu.log
