# seam path with rank-2 chains, multi-process suites after the epoch fix
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --workload lap16k --steps 20 --warmup 5 --no-cpu-baseline --no-check > gpurun_out/bench_lap16k.log 2>&1
tail -1 gpurun_out/bench_lap16k.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('lap16k', round(d['value'],1), round(d['e2e']['value'],1), round(d['e2e']['in_process']['value'],1))" 2>/dev/null || tail -3 gpurun_out/bench_lap16k.log
timeout 2400 python -m pytest tests/test_gpu_ipc.py tests/test_gpu_integration.py tests/test_gpu_rescale3d.py tests/test_gpu_temporal.py -q -p no:cacheprovider --timeout 900 -rfE > gpurun_out/mp_tests.log 2>&1; echo "rc=$?"; tail -4 gpurun_out/mp_tests.log
