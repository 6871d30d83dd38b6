# in-order est_tb default: parity suites + bench; warm-spare restarts; C5; IPC host profile
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_temporal.py tests/test_gpu_bench_configs.py tests/test_gpu_integration.py tests/test_gpu_hash.py -q -p no:cacheprovider --timeout 1200 -rfE -s > gpurun_out/v3_tests.log 2>&1; echo "rc=$?" >> gpurun_out/v3_tests.log
grep -E "warm restart|passed|failed" gpurun_out/v3_tests.log | tail -5
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c4.log 2>&1; tail -1 gpurun_out/bench_c4.log | cut -c1-250
timeout 900 python bench.py --workload c2 --steps 40 --warmup 5 > gpurun_out/bench_c2.log 2>&1; tail -1 gpurun_out/bench_c2.log | cut -c1-250
: > gpurun_out/c2sweep.log
for cfg in "EST_TB_MIN_ITEMS=4096" "EST_TB_MIN_ITEMS=1024" "EST_TB_PREFETCH=4" "EST_TB_MIN_ITEMS=3072 EST_TB_PREFETCH=4"; do
  echo "== c2 $cfg" >> gpurun_out/c2sweep.log
  env $cfg timeout 300 python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu-baseline --no-check > gpurun_out/sweep_one.log 2>&1
  tail -1 gpurun_out/sweep_one.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['kernel_ms'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> gpurun_out/c2sweep.log 2>&1 || tail -3 gpurun_out/sweep_one.log >> gpurun_out/c2sweep.log
done
for cfg in "EST_TB_PREFETCH=4" "EST_TB_ZCHUNK=128 EST_TB_PREFETCH=4"; do
  echo "== c4 $cfg" >> gpurun_out/c2sweep.log
  env $cfg timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-check > gpurun_out/sweep_one.log 2>&1
  tail -1 gpurun_out/sweep_one.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['kernel_ms'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> gpurun_out/c2sweep.log 2>&1 || tail -3 gpurun_out/sweep_one.log >> gpurun_out/c2sweep.log
done
cat gpurun_out/c2sweep.log
timeout 1500 python scripts/rescale3d_bench.py > gpurun_out/c5_3d.json 2> gpurun_out/c5_3d.err; echo "c5 rc=$?"; tail -c 1800 gpurun_out/c5_3d.json
timeout 600 python scripts/ipc_host_profile.py > gpurun_out/ipc_prof.log 2>&1; head -30 gpurun_out/ipc_prof.log
