cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_ipc.py tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 300 -k "ipc or multi_tile or large_2d" > gpurun_out/pytest_ov2.log 2>&1; echo rc=$?; tail -2 gpurun_out/pytest_ov2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29577 bench.py --gpus 2 --workload c3 --steps 3 --warmup 3 > gpurun_out/bench_c3_n2.log 2>&1; echo c3n2 rc=$?; tail -1 gpurun_out/bench_c3_n2.log | cut -c1-200
