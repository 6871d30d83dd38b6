#!/bin/bash
# tb chains with B written only by the last chain of a run (EST_TB_SKIPB=1)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_temporal.py -x -q -k "tb" > gpurun_out/tb_tests.log 2>&1
echo "tb tests rc=$?"; tail -2 gpurun_out/tb_tests.log
run() {  # label, env...
  local label=$1; shift
  env "$@" timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/tbs.json 2> gpurun_out/tbs.err
  python -c "
import json; d=json.loads(open('gpurun_out/tbs.json').read().strip().splitlines()[-1])
print('$label', round(d['value'],1), 'kernel', d['roofline']['kernel'], round(d['roofline']['kernel_ms'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 gpurun_out/tbs.err
}
run "ws2 (default)"
run "tb K2 skipB" EST_TB=1
run "tb K2 writeB" EST_TB=1 EST_TB_SKIPB=0
run "tb K4 skipB" EST_TB=1 EST_TB_K=4
run "tb K2 skipB warp R2" EST_TB=1 EST_TB_VARIANT=warp EST_TB_R=2
run "tb K2 skipB prefetch4" EST_TB=1 EST_TB_PREFETCH=4
run "tb K2 skipB 64x22 rpt4" EST_TB=1 EST_TB_BY=22 EST_TB_RPT=4
