cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/c5_scratch
timeout 1200 python -m pytest tests/test_gpu_integration.py tests/test_gpu_ipc.py -q -p no:cacheprovider --timeout 600 > gpurun_out/pytest_integ.log 2>&1; echo "integ rc=$?"; tail -3 gpurun_out/pytest_integ.log
timeout 900 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --workload c2 > gpurun_out/bench_2proc.log 2>&1; echo "2proc rc=$?"; tail -1 gpurun_out/bench_2proc.log | cut -c1-200
EST_SCRATCH=$GRAFT_REPO_ROOT/gpurun_out/c5_scratch timeout 2400 python scripts/rescale_bench.py --n 32768 --iters 100 --workers 8 > gpurun_out/rescale_c5_32k.log 2>&1; echo "rescale32k rc=$?"; tail -1 gpurun_out/rescale_c5_32k.log | cut -c1-1200
grep -h "restore:\|migrate " gpurun_out/c5_scratch/logs/gpu-worker-*.log | sort | head -40
rm -f gpurun_out/c5_scratch/*.dat
