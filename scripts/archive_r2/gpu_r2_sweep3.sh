# tb chain kernel v2c (crossed W/E per half-warp, optional hoisted loads): parity, C4 sweep
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_temporal.py tests/test_gpu_hash.py -q -x -p no:cacheprovider --timeout 600 > gpurun_out/tb_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tb_tests.log; tail -3 gpurun_out/tb_tests.log
: > gpurun_out/sweep.log
for cfg in "EST_TB_HOIST=0" "EST_TB_HOIST=1" "EST_TB_RPT=3" "EST_TB_RPT=3 EST_TB_HOIST=1" "EST_TB_BY=24 EST_TB_HOIST=1" "EST_TB_BY=24" "EST_TB_K=4 EST_TB_BX=32 EST_TB_BY=32" "EST_TB_BX=48 EST_TB_BY=32 EST_TB_RPT=3"; do
  echo "== $cfg" >> gpurun_out/sweep.log
  env $cfg timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/sweep_one.log 2>&1
  tail -1 gpurun_out/sweep_one.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['kernel_ms'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> gpurun_out/sweep.log 2>&1 || tail -3 gpurun_out/sweep_one.log >> gpurun_out/sweep.log
done
cat gpurun_out/sweep.log
