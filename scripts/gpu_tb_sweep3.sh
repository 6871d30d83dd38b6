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
run "zc171" EST_TB_ZCHUNK=171
run "zc192" EST_TB_ZCHUNK=192
run "zc205" EST_TB_ZCHUNK=205
run "zc256" EST_TB_ZCHUNK=256
run "zc146" EST_TB_ZCHUNK=146
run "default again"
run "zc171 again" EST_TB_ZCHUNK=171
run "zc192 again" EST_TB_ZCHUNK=192
