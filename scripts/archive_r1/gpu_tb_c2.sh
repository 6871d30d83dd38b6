#!/bin/bash
# tb vs ws2 at C2 (512^3): z-chunk choices (EST_TB_MIN_POINTS=0 forces chains)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
run() {
  local label=$1; shift
  env "$@" timeout 600 python bench.py --workload c2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/tbs.json 2> gpurun_out/tbs.err
  python -c "
import json; d=json.loads(open('gpurun_out/tbs.json').read().strip().splitlines()[-1])
print('$label', round(d['value'],1), d['roofline']['kernel'], round(d['roofline']['kernel_ms'],4), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/tbs.err
}
run "ws2 (default)"
for zc in 32 48 64 96 128 170 255; do run "tb zc$zc" EST_TB_MIN_POINTS=0 EST_TB_ZCHUNK=$zc; done
run "tb 64x28 zc64" EST_TB_MIN_POINTS=0 EST_TB_BX=64 EST_TB_BY=28 EST_TB_ZCHUNK=64
run "ws2 again"
