cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_temporal.py -q -p no:cacheprovider --timeout 300 -x > gpurun_out/pytest_tb.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tb.log; tail -15 gpurun_out/pytest_tb.log
timeout 600 python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_tb.log 2>&1; echo "c4 rc=$?"; tail -1 gpurun_out/bench_c4_tb.log | cut -c1-300
for cfg in "64 16 2 2" "64 16 3 2" "64 8 2 2" "128 8 2 2" "64 16 2 3" "32 16 2 2" "64 32 4 2"; do
  set -- $cfg
  EST_TB_BX=$1 EST_TB_BY=$2 EST_TB_RPT=$3 EST_TB_PREFETCH=$4 timeout 600 python bench.py --workload c4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/c4tb_$1_$2_$3_$4.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/c4tb_$1_$2_$3_$4.log').read().strip().splitlines()[-1]); print('c4 tb bx=$1 by=$2 rpt=$3 p=$4', round(d['value'],1), round(d['roofline']['frac'],3), round(d['roofline']['kernel_ms'],3), d['clocks']['sm_mhz'])" 2>&1 | tail -1
done
