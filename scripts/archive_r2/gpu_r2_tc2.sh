# est_tc parity suite + config sweep (C3 wave, paper-shape Laplace) + e2e probe
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_temporal2d.py -q -p no:cacheprovider --timeout 600 -rfE > gpurun_out/tc_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tc_tests.log; tail -5 gpurun_out/tc_tests.log
EST_TC_VEC=8 timeout 1200 python -m pytest tests/test_gpu_temporal2d.py -q -p no:cacheprovider --timeout 600 -rfE > gpurun_out/tc_tests8.log 2>&1; echo "rc=$?" >> gpurun_out/tc_tests8.log; tail -3 gpurun_out/tc_tests8.log
for cfg in "c3 EST_TC_VEC=16" "c3 EST_TC_VEC=8" "c3 EST_TC_VEC=8 EST_TC_RB=10" "c3 EST_TC_VEC=8 EST_TC_PREFETCH=1" "c3 EST_TC_VEC=8 EST_TC_PREFETCH=3" "c3 EST_TC_VEC=16 EST_TC_RB=10" "c3 EST_TC_VEC=8 EST_TC_YCHUNK=256" "lap16k EST_TC_RB=6" "lap16k EST_TC_PREFETCH=1" "lap16k EST_TC_PREFETCH=3" "lap16k EST_TC_RB=9"; do
  set -- $cfg; wl=$1; shift
  echo "== $wl $*"
  env "$@" timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --no-seam --no-check > gpurun_out/tc_bench.log 2>&1
  tail -1 gpurun_out/tc_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['roofline']['kernel'], round(d['roofline']['kernel_ms'],3), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'], round(d['e2e']['value'],1))" || tail -20 gpurun_out/tc_bench.log
done
for wl in c4 lap16k; do timeout 600 python scripts/e2e_probe.py $wl 16 > gpurun_out/e2e_probe_$wl.log 2>&1; cat gpurun_out/e2e_probe_$wl.log | tail -18; done
