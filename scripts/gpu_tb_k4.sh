#!/bin/bash
# K = 4 chains on C4 (4 B/LUP) vs the K = 2 default; parity of K = 4 first
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
EST_TB_K=4 EST_TB_BX=32 EST_TB_BY=32 timeout 900 python -m pytest tests/test_gpu_temporal.py -x -q -k "tb and not warp" > gpurun_out/k4_tests.log 2>&1
echo "k4 tests rc=$?"; tail -2 gpurun_out/k4_tests.log
run() {
  local label=$1; shift
  env "$@" timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/tbs.json 2> gpurun_out/tbs.err
  python -c "
import json; d=json.loads(open('gpurun_out/tbs.json').read().strip().splitlines()[-1])
print('$label', round(d['value'],1), d['roofline']['kernel'], round(d['roofline']['kernel_ms'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/tbs.err
}
run "K2 48x32 default"
run "K4 32x32 pf2" EST_TB_K=4 EST_TB_BX=32 EST_TB_BY=32
run "K4 32x32 pf1" EST_TB_K=4 EST_TB_BX=32 EST_TB_BY=32 EST_TB_PREFETCH=1
run "K4 32x30 pf1" EST_TB_K=4 EST_TB_BX=32 EST_TB_BY=30 EST_TB_PREFETCH=1
run "K4 24x32 pf2" EST_TB_K=4 EST_TB_BX=24 EST_TB_BY=32
