cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_bench.py tests/test_gpu_temporal.py -q -p no:cacheprovider --timeout 900 > gpurun_out/pytest_misc.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_misc.log
