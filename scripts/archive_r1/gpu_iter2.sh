cd $GRAFT_REPO_ROOT
timeout 600 python scripts/debug_stream.py rand3d > gpurun_out/debug_stream.log 2>&1; echo "rc=$?" >> gpurun_out/debug_stream.log
tail -3 gpurun_out/debug_stream.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for cfg in "16 8 4" "16 4 4" "16 8 2" "32 8 2" "8 8 4" "16 16 4"; do
  set -- $cfg
  EST_STREAM_BY=$1 EST_STREAM_TY=$2 EST_STREAM_PREFETCH=$3 timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_sweep_$1_$2_$3.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_sweep_$1_$2_$3.log').read().strip().splitlines()[-1]); print('BY=$1 TY=$2 P=$3', round(d['value'],1), round(d['roofline']['frac'],3), round(d['roofline']['kernel_ms'],3))" 2>&1 | tail -1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:est_stream -s 3 -c 1 -o gpurun_out/prof_c4_stream3 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
