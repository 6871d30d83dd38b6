# non-persistent est_tb sweep (C4, C2) + ncu of the non-persistent C4 launch
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/np.log
for wl in c4 c2; do
for cfg in "EST_TB_PERSISTENT=0 EST_TB_ZCHUNK=48" "EST_TB_PERSISTENT=0 EST_TB_ZCHUNK=64" "EST_TB_PERSISTENT=0 EST_TB_ZCHUNK=96" "EST_TB_PERSISTENT=0 EST_TB_ZCHUNK=128" "EST_TB_PERSISTENT=0 EST_TB_ZCHUNK=256" "EST_TB_PERSISTENT=0 EST_TB_ZCHUNK=96 EST_TB_BY=24" "EST_TB_PERSISTENT=0 EST_TB_ZCHUNK=96 EST_TB_PREFETCH=3"; do
  echo "== $wl $cfg" >> gpurun_out/np.log
  env $cfg EST_TB_MIN_POINTS=0 timeout 300 python bench.py --workload $wl --steps 8 --warmup 3 --no-cpu-baseline --no-check > gpurun_out/sweep_one.log 2>&1
  tail -1 gpurun_out/sweep_one.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['kernel_ms'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> gpurun_out/np.log 2>&1 || tail -3 gpurun_out/sweep_one.log >> gpurun_out/np.log
done
done
cat gpurun_out/np.log
EST_TB_PERSISTENT=0 EST_TB_ZCHUNK=96 bash scripts/ncu_kernel.sh c4 est_tb r2_c4_tb_np96
