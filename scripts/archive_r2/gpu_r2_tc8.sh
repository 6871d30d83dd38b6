# est_tc: P from HBM into registers a stage ahead (pglobal) vs TMA-staged P; parity + C3 sweep
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in 16 8; do
EST_TC_VEC=$v timeout 1200 python -m pytest tests/test_gpu_temporal2d.py -q -p no:cacheprovider --timeout 600 -rfE > gpurun_out/tc_tests$v.log 2>&1; echo "vec $v rc=$?"; tail -2 gpurun_out/tc_tests$v.log
done
for cfg in "c3 EST_TC_VEC=8 EST_TC_PREFETCH=1 EST_TC_RB=5" "c3 EST_TC_VEC=8 EST_TC_PREFETCH=2 EST_TC_RB=5" "c3 EST_TC_VEC=8 EST_TC_PREFETCH=3 EST_TC_RB=5" "c3 EST_TC_VEC=8 EST_TC_PREFETCH=4 EST_TC_RB=5" "c3 EST_TC_VEC=8 EST_TC_PREFETCH=2 EST_TC_RB=4" "c3 EST_TC_VEC=8 EST_TC_PREFETCH=3 EST_TC_RB=4" "c3 EST_TC_VEC=16 EST_TC_PREFETCH=2 EST_TC_RB=5" "c3 EST_TC_VEC=8 EST_TC_PREFETCH=1 EST_TC_RB=5 EST_TC_PGLOBAL=0"; do
  set -- $cfg; wl=$1; shift
  echo "== $wl $*"
  env "$@" timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --no-seam --no-check > gpurun_out/tc_bench.log 2>&1
  tail -1 gpurun_out/tc_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['roofline']['kernel'], round(d['roofline']['kernel_ms'],3), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'], round(d['e2e']['value'],1))" 2>/dev/null || grep -m2 Error gpurun_out/tc_bench.log
done
