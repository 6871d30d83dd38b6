#!/bin/bash
# tb 48x32: persistence, z-chunk, L2 promotion (C4)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
run() {
  local label=$1; shift
  env "$@" timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/tbs.json 2> gpurun_out/tbs.err
  python -c "
import json; d=json.loads(open('gpurun_out/tbs.json').read().strip().splitlines()[-1])
print('$label', round(d['value'],1), d['roofline']['kernel'], round(d['roofline']['kernel_ms'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/tbs.err
}
run "default"
run "48x16 minb2" EST_TB_BX=48 EST_TB_BY=16 EST_TB_MINB=2
run "48x16" EST_TB_BX=48 EST_TB_BY=16
run "32x16 minb3" EST_TB_BX=32 EST_TB_BY=16 EST_TB_MINB=3
run "32x22 minb2" EST_TB_BX=32 EST_TB_BY=22 EST_TB_MINB=2
run "default again"
