#!/bin/bash
# mbarrier try_wait suspend-time hint: C4 (tb / ws2), C3
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
run() {
  local label=$1 w=$2; shift 2
  env "$@" timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/w.json 2> gpurun_out/w.err
  python -c "
import json; d=json.loads(open('gpurun_out/w.json').read().strip().splitlines()[-1])
print('$label', round(d['value'],1), d['roofline']['kernel'], round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 gpurun_out/w.err
}
for h in 0 200 1000 5000 20000; do run "c4 tb hint=$h" c4 EST_WAIT_HINT_NS=$h; done
for h in 0 1000 20000; do run "c4 ws2 hint=$h" c4 EST_TB=0 EST_WAIT_HINT_NS=$h; done
for h in 0 1000; do run "c3 hint=$h" c3 EST_WAIT_HINT_NS=$h; done
