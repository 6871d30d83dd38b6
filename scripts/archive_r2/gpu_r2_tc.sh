# rank-2 two-sweep chains (est_tc): parity suite, C3 / paper-shape Laplace benches vs single sweeps, e2e probe
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_temporal2d.py -x -q -p no:cacheprovider --timeout 600 -rfE > gpurun_out/tc_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tc_tests.log; tail -25 gpurun_out/tc_tests.log
for cfg in "c3" "c3 EST_TC=0" "lap16k" "lap16k EST_TC=0"; do
  set -- $cfg; wl=$1; shift
  echo "== $wl $*"
  env "$@" timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --no-seam > gpurun_out/tc_bench.log 2>&1
  tail -1 gpurun_out/tc_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['roofline']['kernel'], round(d['roofline']['kernel_ms'],3), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'], d.get('check',{}).get('ok'), round(d['e2e']['value'],1))" || tail -20 gpurun_out/tc_bench.log
done
timeout 600 python scripts/e2e_probe.py c4 > gpurun_out/e2e_probe.log 2>&1; tail -3 gpurun_out/e2e_probe.log
