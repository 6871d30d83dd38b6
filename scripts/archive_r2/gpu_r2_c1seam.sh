cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --workload c1 --no-cpu-baseline > gpurun_out/bench_c1.log 2>&1; tail -1 gpurun_out/bench_c1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1', round(d['value'],1), round(d['e2e']['value'],1), round(d['e2e']['in_process']['value'],1), d['check']['ok'])"
timeout 1500 python -m pytest tests/test_gpu_resident_smem.py tests/test_gpu_integration.py tests/test_gpu_reference_suites.py -q -p no:cacheprovider --timeout 1400 -rfE > gpurun_out/c1seam_tests.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/c1seam_tests.log
