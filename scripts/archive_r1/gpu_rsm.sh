#!/bin/bash
# resident-smem: parity, then C1 bench over KM / rows-per-thread / threads
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
[ -n "$RSM_TESTS" ] && timeout 900 python -m pytest tests/test_gpu_resident_smem.py -x -q > gpurun_out/rsm_tests.log 2>&1
echo "rsm tests rc=$?"; tail -3 gpurun_out/rsm_tests.log
for cfg in "10 10 1024" "10 12 1024" "10 16 1024" "12 12 1024" "12 16 1024" "10 16 512" "12 10 1024"; do
  set -- $cfg
  EST_RSM_K=$1 EST_RSM_RPT=$2 EST_RSM_THREADS=$3 timeout 300 python bench.py --workload c1 --no-cpu-baseline > gpurun_out/rsm_c1.json 2>gpurun_out/rsm_c1.err
  python -c "
import json; d=json.loads(open('gpurun_out/rsm_c1.json').read().strip().splitlines()[-1])
print('K=$1 RPT=$2 NT=$3', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'launches', d['gpu_launches'], d['roofline']['kernel'])" || tail -5 gpurun_out/rsm_c1.err
done
EST_RESIDENT_SMEM=0 timeout 300 python bench.py --workload c1 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('rsm off', round(d['value'],1))"
