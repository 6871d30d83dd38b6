cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 300 -x > gpurun_out/pytest_2d.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_2d.log; tail -4 gpurun_out/pytest_2d.log
for cfg in "128 16 4 3" "128 32 8 3" "128 8 4 3" "64 32 8 3" "128 16 4 2" "128 16 8 4" "248 8 4 3"; do
  set -- $cfg
  EST_STREAM2D_BX=$1 EST_STREAM2D_BY=$2 EST_STREAM2D_TY=$3 EST_STREAM2D_PREFETCH=$4 timeout 600 python bench.py --workload c3 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/c3_$1_$2_$3_$4.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/c3_$1_$2_$3_$4.log').read().strip().splitlines()[-1]); print('c3 bx=$1 by=$2 ty=$3 p=$4', round(d['value'],1), round(d['roofline']['frac'],3), round(d['roofline']['kernel_ms'],3))" 2>&1 | tail -1
done
timeout 600 python bench.py --workload c1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1.log 2>&1; tail -1 gpurun_out/bench_c1.log
