cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/last
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/last/smoke.log 2>&1; echo "smoke rc=$?"
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1500 -rfE > gpurun_out/last/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/last/pytest_gpu.log
tail -4 gpurun_out/last/pytest_gpu.log
