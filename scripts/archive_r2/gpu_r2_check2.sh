# round-2 re-entry checkpoint: slab-chain tests first, benches (1/2/4 ranks), then the full GPU suite
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
(nproc; lscpu | grep -E 'Model name|^CPU\(s\)'; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv) > gpurun_out/box_info.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_temporal.py tests/test_gpu_ipc.py -q -p no:cacheprovider --timeout 600 -rfE > gpurun_out/slab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/slab_tests.log; tail -8 gpurun_out/slab_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log; tail -4 gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c4.log 2>&1; tail -1 gpurun_out/bench_c4.log | cut -c1-400
for n in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n bench.py --gpus $n --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${n}r.log 2>&1; tail -1 gpurun_out/bench_${n}r.log | cut -c1-400
done
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rfE > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
