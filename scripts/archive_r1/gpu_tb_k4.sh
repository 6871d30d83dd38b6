#!/bin/bash
# K = 4 chains on C4 (4 B/LUP) vs the K = 2 default, after the padded-z fix
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
run() {
  local label=$1; shift
  env "$@" timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/tbs.json 2> gpurun_out/tbs.err
  python -c "
import json; d=json.loads(open('gpurun_out/tbs.json').read().strip().splitlines()[-1])
print('$label', round(d['value'],1), d['roofline']['kernel'], round(d['roofline']['kernel_ms'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/tbs.err
}
run "K2 default"
for cfg in "32 32 2" "32 30 2" "24 32 2" "32 26 1" "40 24 2"; do
  set -- $cfg
  run "K4 ${1}x${2} pf$3" EST_TB_VALIDATED_K=2,4 EST_TB_K=4 EST_TB_BX=$1 EST_TB_BY=$2 EST_TB_PREFETCH=$3
done
run "K2 again"
