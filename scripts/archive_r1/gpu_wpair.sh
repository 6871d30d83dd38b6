#!/bin/bash
# wave pairs (EST_WPAIR=1): parity, then C3 bench over tile shapes
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wavepair.py -x -q > gpurun_out/wp_tests.log 2>&1
echo "wp tests rc=$?"; tail -3 gpurun_out/wp_tests.log
run() {
  local label=$1; shift
  env "$@" timeout 300 python bench.py --workload c3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/wp.json 2>gpurun_out/wp.err
  python -c "
import json; d=json.loads(open('gpurun_out/wp.json').read().strip().splitlines()[-1])
print('$label', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['roofline']['kernel'], round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],3))" || tail -3 gpurun_out/wp.err
}
run "ws2 default"
for cfg in "128 32 256" "128 32 512" "64 32 256" "128 16 256" "256 16 256" "64 64 256" "128 64 512"; do
  set -- $cfg
  run "wpair ${1}x${2} nt$3" EST_WPAIR=1 EST_WPAIR_TX=$1 EST_WPAIR_TY=$2 EST_WPAIR_THREADS=$3
done
