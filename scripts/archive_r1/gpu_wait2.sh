#!/bin/bash
# back-off between unsuccessful mbarrier tries (EST_WAIT_SLEEP_NS)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
run() {
  local label=$1 w=$2; shift 2
  env "$@" timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/w.json 2> gpurun_out/w.err
  python -c "
import json; d=json.loads(open('gpurun_out/w.json').read().strip().splitlines()[-1])
print('$label', round(d['value'],1), d['roofline']['kernel'], round(d['roofline']['kernel_ms'],4), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/w.err
}
for ns in 0 20 64 200 0; do run "c4 tb sleep=$ns" c4 EST_WAIT_SLEEP_NS=$ns; done
for ns in 0 64; do run "c4 ws2 sleep=$ns" c4 EST_TB=0 EST_WAIT_SLEEP_NS=$ns; done
for ns in 0 64; do run "c3 sleep=$ns" c3 EST_WAIT_SLEEP_NS=$ns; done
