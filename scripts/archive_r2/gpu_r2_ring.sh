cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
EST_TC_RING=1 timeout 1200 python -m pytest tests/test_gpu_temporal2d.py -q -p no:cacheprovider --timeout 600 -rfE > gpurun_out/ring_tests.log 2>&1; echo "ring1 tests rc=$?"; tail -2 gpurun_out/ring_tests.log
for cfg in "lap16k EST_TC_RING=0" "lap16k EST_TC_RING=1" "lap16k EST_TC_RING=1 EST_TC_PREFETCH=2" "lap16k EST_TC_RING=0" "lap16k EST_TC_RING=1" "c3 EST_TC_ROT=1 EST_TC_RING=1" "c3 EST_TC_ROT=1 EST_TC_RING=0"; do
  set -- $cfg; wl=$1; shift
  echo "== $wl $*"
  env "$@" timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --no-seam --no-check > gpurun_out/tc_bench.log 2>&1
  tail -1 gpurun_out/tc_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['kernel_ms'],3), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" 2>/dev/null || grep -m2 Error gpurun_out/tc_bench.log
done
