cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for wl in c1 c4; do timeout 900 python bench.py --workload $wl --no-cpu-baseline --no-check > gpurun_out/bench_$wl.log 2>&1; tail -1 gpurun_out/bench_$wl.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$wl', round(d['value'],1), round(d['e2e']['value'],1), round(d['e2e']['in_process']['value'],1))"; done
timeout 2000 python -m pytest tests/test_gpu_integration.py tests/test_gpu_reference_suites.py tests/test_gpu_rescale3d.py tests/test_gpu_ipc.py -q -p no:cacheprovider --timeout 1500 -rfE > gpurun_out/graphseam_tests.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/graphseam_tests.log
