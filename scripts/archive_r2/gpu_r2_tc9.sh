# est_tc final defaults: parity suites (tc + bench-size lap16k), benches, ncu of the shipped est_tc
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_temporal2d.py tests/test_gpu_resident_smem.py -q -p no:cacheprovider --timeout 600 -rfE > gpurun_out/tc_tests.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/tc_tests.log
timeout 1500 python -m pytest tests/test_gpu_bench_configs.py -q -p no:cacheprovider --timeout 1400 -rfE -k "lap16k or c3" > gpurun_out/tc_cfg_tests.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/tc_cfg_tests.log
for wl in lap16k c3; do
  timeout 900 python bench.py --workload $wl --steps 20 --warmup 5 > gpurun_out/bench_$wl.log 2>&1
  tail -1 gpurun_out/bench_$wl.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$wl', round(d['value'],1), d['roofline']['kernel'], round(d['roofline']['kernel_ms'],3), round(d['roofline']['frac'],3), d['clocks'], d['check']['ok'], round(d['e2e']['value'],1))" 2>/dev/null || tail -3 gpurun_out/bench_$wl.log
done
bash scripts/ncu_kernel.sh lap16k est_tc r2_lap16k_tc_final
