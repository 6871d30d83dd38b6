cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_ipc.py tests/test_gpu_integration.py "tests/test_gpu_parity.py::test_golden_case_multi_tile" -q -p no:cacheprovider --timeout 300 -x > gpurun_out/pytest_overlap.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_overlap.log; tail -4 gpurun_out/pytest_overlap.log
timeout 900 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 1 --workload c2 > gpurun_out/bench_2proc.log 2>&1; tail -1 gpurun_out/bench_2proc.log
timeout 1500 python scripts/rescale_bench.py --n 16384 --iters 100 --workers 8 > gpurun_out/rescale_c5.log 2>&1; tail -2 gpurun_out/rescale_c5.log
