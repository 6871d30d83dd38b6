# est_tc with 8-byte vectors (16-byte aligned TMA box starts): parity + C3 sweep
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
EST_TC_VEC=8 timeout 1200 python -m pytest tests/test_gpu_temporal2d.py -q -p no:cacheprovider --timeout 600 -rfE > gpurun_out/tc_tests8.log 2>&1; echo "vec 8 rc=$?"; tail -2 gpurun_out/tc_tests8.log
for cfg in "c3 EST_TC_VEC=8" "c3 EST_TC_VEC=8 EST_TC_PREFETCH=1" "c3 EST_TC_VEC=8 EST_TC_PREFETCH=3" "c3 EST_TC_VEC=8 EST_TC_YCHUNK=1024" "c3 EST_TC_VEC=8 EST_TC_RB=10" "lap16k EST_TC_VEC=8"; do
  set -- $cfg; wl=$1; shift
  echo "== $wl $*"
  env "$@" timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --no-seam --no-check > gpurun_out/tc_bench.log 2>&1
  tail -1 gpurun_out/tc_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['roofline']['kernel'], round(d['roofline']['kernel_ms'],3), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'], round(d['e2e']['value'],1))" 2>/dev/null || grep -m2 Error gpurun_out/tc_bench.log
done
