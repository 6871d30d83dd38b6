# est_tb prefetch depth, alternating to control for clocks
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in "c4 EST_TB_PREFETCH=3" "c4 EST_TB_PREFETCH=4" "c4 EST_TB_PREFETCH=5" "c4 EST_TB_PREFETCH=3" "c4 EST_TB_PREFETCH=4" "c4 EST_TB_PREFETCH=5" "c4 EST_TB_PREFETCH=4 EST_TB_ZCHUNK=128" "c2 EST_TB_PREFETCH=3" "c2 EST_TB_PREFETCH=4" "c2 EST_TB_PREFETCH=5"; do
  set -- $cfg; wl=$1; shift
  echo "== $wl $*"
  env "$@" timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --no-seam --no-check > gpurun_out/tb_bench.log 2>&1
  tail -1 gpurun_out/tb_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['kernel_ms'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>/dev/null || grep -m2 Error gpurun_out/tb_bench.log
done
