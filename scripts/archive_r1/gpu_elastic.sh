cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/c5_scratch
timeout 1200 python -m pytest tests/test_gpu_integration.py -q -p no:cacheprovider --timeout 600 > gpurun_out/pytest_integ.log 2>&1; echo "integ rc=$?"; tail -2 gpurun_out/pytest_integ.log
EST_SCRATCH=$GRAFT_REPO_ROOT/gpurun_out/c5_scratch timeout 2400 python scripts/rescale_bench.py --n 32768 --iters 100 --workers 8 > gpurun_out/rescale_c5_32k.log 2>&1; echo "rescale32k rc=$?"; tail -1 gpurun_out/rescale_c5_32k.log | cut -c1-1200
grep -h "restore:" gpurun_out/c5_scratch/logs/gpu-worker-*.log | sort | head -20
rm -rf gpurun_out/c5_scratch
