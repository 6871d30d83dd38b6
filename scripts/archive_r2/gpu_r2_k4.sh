# e2e probe (where the seam step time goes) + K=4 chains on C4/C2
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/e2e_probe.py c4 > gpurun_out/e2e_probe.log 2>&1; tail -2 gpurun_out/e2e_probe.log
for cfg in "c4 EST_TB_K=2" "c4 EST_TB_K=4" "c4 EST_TB_K=4 EST_TB_ZCHUNK=192" "c4 EST_TB_K=4 EST_TB_BY=48 EST_TB_ZCHUNK=128" "c2 EST_TB_K=4" "c2 EST_TB_K=4 EST_TB_MIN_ITEMS=1024"; do
  set -- $cfg; wl=$1; shift
  echo "== $wl $*"
  env "$@" timeout 600 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --no-seam --no-check > gpurun_out/k4.log 2>&1
  tail -1 gpurun_out/k4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['kernel_ms'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -5 gpurun_out/k4.log
done
