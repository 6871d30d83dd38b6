cd $GRAFT_REPO_ROOT
rm -rf /tmp/est-r3-*; mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_rescale3d.py tests/test_gpu_integration.py tests/test_gpu_daemon.py -q -p no:cacheprovider --timeout 1500 -rfE > gpurun_out/pool_tests.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/pool_tests.log
timeout 1500 python scripts/rescale3d_bench.py --iters 200 --batches 2 > gpurun_out/c5pool.json 2> gpurun_out/c5pool.err; echo "rc=$?"
python -c "import json; d=json.load(open('gpurun_out/c5pool.json')); print({k: round(v['total_ms']) for k, v in d['rescales'].items()}, d['bit_equal_to_unrescaled'])"
