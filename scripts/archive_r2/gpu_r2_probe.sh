# tb chain kernel: ncu of the default (v2c) and of the no-shared-loads probe; C4 timing of the probe
cd $GRAFT_REPO_ROOT
: > gpurun_out/sweep.log
for cfg in "EST_TB_PROBE=noshared" "EST_TB_PROBE=noshared EST_TB_L2PROMO=0" "EST_TB_L2PROMO=0"; do
  echo "== $cfg" >> gpurun_out/sweep.log
  env $cfg timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-check > gpurun_out/sweep_one.log 2>&1
  tail -1 gpurun_out/sweep_one.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['kernel_ms'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> gpurun_out/sweep.log 2>&1 || tail -3 gpurun_out/sweep_one.log >> gpurun_out/sweep.log
done
cat gpurun_out/sweep.log
bash scripts/ncu_kernel.sh c4 est_tb r2_tb_v2c
bash scripts/ncu_kernel.sh c4 est_tb r2_tb_probe_noshared EST_TB_PROBE=noshared
bash scripts/ncu_kernel.sh c4 est_tb r2_tb_promo0 EST_TB_L2PROMO=0
