cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/crit5_probe.py 1 100 > gpurun_out/crit5.log 2>&1; cat gpurun_out/crit5.log | tail -4
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_c4.log 2>&1; tail -1 gpurun_out/ref_c4.log | cut -c1-400
: > gpurun_out/sweep2.log
for cfg in "EST_TB_ZCHUNK=64" "EST_TB_PERSISTENT=0" "EST_TB_ZCHUNK=96 EST_TB_PERSISTENT=0" "EST_TB_BX=32 EST_TB_BY=32" "EST_TB_BX=128 EST_TB_BY=16"; do
  echo "== $cfg" >> gpurun_out/sweep2.log
  env $cfg timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-check > gpurun_out/sweep_one.log 2>&1
  tail -1 gpurun_out/sweep_one.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['kernel_ms'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> gpurun_out/sweep2.log 2>&1 || tail -3 gpurun_out/sweep_one.log >> gpurun_out/sweep2.log
done
cat gpurun_out/sweep2.log
for wl in c2; do EST_TB=0 timeout 300 python bench.py --workload c2 --steps 20 --warmup 3 --no-cpu-baseline --no-check > gpurun_out/c2_notb.log 2>&1; tail -1 gpurun_out/c2_notb.log | cut -c1-200; done
