# slab chains (multi-tile / multi-process temporal blocking) + seam probe
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_temporal.py tests/test_gpu_ipc.py -q -p no:cacheprovider --timeout 600 -rfE > gpurun_out/slab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/slab_tests.log; tail -8 gpurun_out/slab_tests.log
timeout 600 python scripts/seam_probe.py > gpurun_out/seam_probe.log 2>&1; cat gpurun_out/seam_probe.log | tail -8
for n in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n bench.py --gpus $n --steps 5 --warmup 3 > gpurun_out/bench_${n}r.log 2>&1; tail -1 gpurun_out/bench_${n}r.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($n, 'ranks', round(d['value'],1), d['roofline']['kernel'], round(d['roofline']['kernel_ms'],3), d['clocks']['sm_mhz'])" || tail -5 gpurun_out/bench_${n}r.log
done
