# device-flag IPC protocol: IPC parity tests, host profile, criterion-5 probe, 2-rank bench, seam e2e bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ipc.py -x -q -p no:cacheprovider --timeout 300 > gpurun_out/ipc_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ipc_tests.log; tail -3 gpurun_out/ipc_tests.log
timeout 600 python scripts/ipc_host_profile.py > gpurun_out/ipc_prof.log 2>&1; head -3 gpurun_out/ipc_prof.log
timeout 600 python scripts/crit5_probe.py 1 100 > gpurun_out/crit5.log 2>&1; tail -2 gpurun_out/crit5.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_2r.log 2>&1; tail -1 gpurun_out/bench_2r.log | cut -c1-300
timeout 1800 python -m pytest tests/test_gpu_integration.py tests/test_gpu_reference_suites.py -q -p no:cacheprovider --timeout 1500 -rfE > gpurun_out/integ.log 2>&1; echo "rc=$?" >> gpurun_out/integ.log; tail -5 gpurun_out/integ.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_seam.log 2>&1; tail -1 gpurun_out/bench_c4_seam.log
