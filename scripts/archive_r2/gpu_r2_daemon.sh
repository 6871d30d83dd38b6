cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_daemon.py -q -p no:cacheprovider --timeout 600 -rfE > gpurun_out/daemon_tests.log 2>&1; echo "rc=$?"; tail -15 gpurun_out/daemon_tests.log
