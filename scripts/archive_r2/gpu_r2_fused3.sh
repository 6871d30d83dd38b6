cd $GRAFT_REPO_ROOT
rm -rf /tmp/est-r3-*; mkdir -p gpurun_out
timeout 600 python scripts/debug_fused.py 8 2>&1 | tail -5
timeout 2400 python -m pytest tests/test_gpu_ipc.py tests/test_gpu_rescale3d.py -q -p no:cacheprovider --timeout 900 -rfE > gpurun_out/fused_tests.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/fused_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-seam --no-check > gpurun_out/bench_1r.log 2>&1; tail -1 gpurun_out/bench_1r.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(1, 'rank', round(d['value'],1), round(d['roofline']['kernel_ms'],3), d['clocks']['sm_mhz'])"
for fp in 1 0; do for n in 2 4; do
EST_FUSED_PUSH=$fp timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n bench.py --gpus $n --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${n}r.log 2>&1; tail -1 gpurun_out/bench_${n}r.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fused $fp', $n, 'ranks', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline']['kernel_ms'],3), d['clocks']['sm_mhz'])" || tail -5 gpurun_out/bench_${n}r.log
done; done
EST_WORKER_LOG=1 timeout 1500 python scripts/rescale3d_bench.py --iters 200 --batches 2 > gpurun_out/c5probe.json 2> gpurun_out/c5probe.err; echo "rc=$?"
python -c "import json; d=json.load(open('gpurun_out/c5probe.json')); print(json.dumps(d['rescales']), d['bit_equal_to_unrescaled'], d['glups'])"
