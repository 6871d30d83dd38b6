# est_tc occupancy sweep: stage rows / prefetch / vector width (C3 wave, paper-shape Laplace)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in "c3 EST_TC_VEC=8 EST_TC_PREFETCH=0" "c3 EST_TC_VEC=16 EST_TC_PREFETCH=0" "c3 EST_TC_VEC=8 EST_TC_PREFETCH=1 EST_TC_RB=3" "c3 EST_TC_VEC=8 EST_TC_PREFETCH=2 EST_TC_RB=3" "c3 EST_TC_VEC=8 EST_TC_PREFETCH=1 EST_TC_RB=4" "c3 EST_TC_VEC=16 EST_TC_PREFETCH=1 EST_TC_RB=3" "lap16k EST_TC_PREFETCH=0" "lap16k EST_TC_PREFETCH=1 EST_TC_RB=2" "lap16k EST_TC_PREFETCH=2 EST_TC_RB=2" "lap16k EST_TC_PREFETCH=1 EST_TC_RB=4"; do
  set -- $cfg; wl=$1; shift
  echo "== $wl $*"
  env "$@" timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --no-seam --no-check > gpurun_out/tc_bench.log 2>&1
  tail -1 gpurun_out/tc_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['roofline']['kernel'], round(d['roofline']['kernel_ms'],3), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'], round(d['e2e']['value'],1))" 2>/dev/null || grep -m2 Error gpurun_out/tc_bench.log
done
