#!/bin/bash
# resident-smem with two columns per item (EST_RSM_PAIR=1): parity, C1 sweep
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
EST_RSM_PAIR=1 timeout 900 python -m pytest tests/test_gpu_resident_smem.py -x -q > gpurun_out/pair_tests.log 2>&1
echo "pair tests rc=$?"; tail -2 gpurun_out/pair_tests.log
run() {
  local label=$1; shift
  env "$@" timeout 300 python bench.py --workload c1 --no-cpu-baseline > gpurun_out/p.json 2>gpurun_out/p.err
  python -c "
import json; d=json.loads(open('gpurun_out/p.json').read().strip().splitlines()[-1])
print('$label', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['roofline']['kernel'])" || tail -3 gpurun_out/p.err
}
run "single K10 R12 1024"
for cfg in "12 1024" "8 1024" "6 1024" "4 1024" "8 512" "12 512"; do
  set -- $cfg
  run "pair K10 R$1 NT$2" EST_RSM_PAIR=1 EST_RSM_RPT=$1 EST_RSM_THREADS=$2
done
run "pair K12 R6 1024" EST_RSM_PAIR=1 EST_RSM_K=12 EST_RSM_RPT=6
