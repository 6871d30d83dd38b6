# main after the chain write-after-read ordering fix: multi-process / slab-chain suites, benches
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/order
timeout 2400 python -m pytest tests/test_gpu_ipc.py tests/test_gpu_rescale3d.py tests/test_gpu_temporal.py tests/test_gpu_integration.py tests/test_gpu_bench_configs.py -q -p no:cacheprovider --timeout 1500 -rfE > gpurun_out/order/tests.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/order/tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/order/bench_c4.log 2>&1; tail -1 gpurun_out/order/bench_c4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4', round(d['value'],1), round(d['e2e']['value'],1), d['clocks']['sm_mhz'], d['check']['ok'])"
for n in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n bench.py --gpus $n --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/order/bench_c4_${n}r.log 2>&1; tail -1 gpurun_out/order/bench_c4_${n}r.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($n, 'ranks', round(d['value'],1), round(d['e2e']['value'],1), d['clocks']['sm_mhz'])" || tail -5 gpurun_out/order/bench_c4_${n}r.log
done
