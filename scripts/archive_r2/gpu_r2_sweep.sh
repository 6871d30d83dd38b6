# tb chain kernel: parity suite, then a C4 config sweep, then ncu of the default
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_temporal.py -q -x -p no:cacheprovider --timeout 600 > gpurun_out/tb_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tb_tests.log; tail -3 gpurun_out/tb_tests.log
for cfg in "EST_TB_PREFETCH=2" "EST_TB_PREFETCH=3" "EST_TB_PREFETCH=5" "EST_TB_BY=16 EST_TB_PREFETCH=3" "EST_TB_BY=16 EST_TB_PREFETCH=5" "EST_TB_RPT=4 EST_TB_PREFETCH=3" "EST_TB_PREFETCH=3 EST_TB_ZCHUNK=128" "EST_TB_PREFETCH=3 EST_TB_L2PROMO=3"; do
  echo "== $cfg" >> gpurun_out/sweep.log
  env $cfg timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['kernel_ms'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> gpurun_out/sweep.log 2>&1
done
cat gpurun_out/sweep.log
env EST_TB_PREFETCH=3 bash scripts/ncu_kernel.sh c4 est_tb r2_tb_v2
