cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in "c4 EST_TB_L2PROMO=2" "c4 EST_TB_L2PROMO=0" "c4 EST_TB_L2PROMO=1" "c4 EST_TB_L2PROMO=3" "c4 EST_TB_L2PROMO=2" "c4 EST_TB_L2PROMO=0"; do
  set -- $cfg; wl=$1; shift
  echo "== $wl $*"
  env "$@" timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --no-seam --no-check > gpurun_out/pr.log 2>&1
  tail -1 gpurun_out/pr.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['kernel_ms'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>/dev/null || grep -m2 Error gpurun_out/pr.log
done
EST_TB_L2PROMO=0 bash scripts/ncu_kernel.sh c4 est_tb r2_c4_tb_promo0
