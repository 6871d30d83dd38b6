# K = 4 chains with the in-order vector-wide est_tb (smaller tiles so three rings fit)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in "c4 EST_TB_K=2" "c4 EST_TB_K=4 EST_TB_BX=32 EST_TB_BY=32" "c4 EST_TB_K=4 EST_TB_BX=64 EST_TB_BY=16" "c4 EST_TB_K=4 EST_TB_BX=32 EST_TB_BY=32 EST_TB_PREFETCH=2" "c4 EST_TB_K=4 EST_TB_BX=48 EST_TB_BY=24" "c2 EST_TB_K=4 EST_TB_BX=32 EST_TB_BY=32"; do
  set -- $cfg; wl=$1; shift
  echo "== $wl $*"
  env "$@" timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --no-seam --no-check > gpurun_out/k4.log 2>&1
  tail -1 gpurun_out/k4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['roofline']['kernel'], round(d['roofline']['kernel_ms'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>/dev/null || grep -m2 Error gpurun_out/k4.log
done
