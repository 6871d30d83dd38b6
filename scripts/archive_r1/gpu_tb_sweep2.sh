#!/bin/bash
# tb (skip-B) geometry sweep on C4
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
run() {  # label, env...
  local label=$1; shift
  env EST_TB=1 "$@" timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/tbs.json 2> gpurun_out/tbs.err
  python -c "
import json; d=json.loads(open('gpurun_out/tbs.json').read().strip().splitlines()[-1])
print('$label', round(d['value'],1), d['roofline']['kernel'], round(d['roofline']['kernel_ms'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/tbs.err
}
run "48x32 r2" EST_TB_BX=48 EST_TB_BY=32
run "56x32 r2" EST_TB_BX=56 EST_TB_BY=32
run "64x28 r2" EST_TB_BX=64 EST_TB_BY=28
run "48x36 r2" EST_TB_BX=48 EST_TB_BY=36
run "40x40 r2" EST_TB_BX=40 EST_TB_BY=40
run "48x46 r3" EST_TB_BX=48 EST_TB_BY=46 EST_TB_RPT=3
run "64x46 r4 pf1" EST_TB_BX=64 EST_TB_BY=46 EST_TB_RPT=4 EST_TB_PREFETCH=1
run "96x30 r4 pf1" EST_TB_BX=96 EST_TB_BY=30 EST_TB_RPT=4 EST_TB_PREFETCH=1
run "64x30 r4" EST_TB_BX=64 EST_TB_BY=30 EST_TB_RPT=4
run "48x30 r2" EST_TB_BX=48 EST_TB_BY=30
run "48x32 r2 zc256" EST_TB_BX=48 EST_TB_BY=32 EST_TB_ZCHUNK=256
