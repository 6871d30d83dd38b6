#!/bin/bash
# resident-smem default on: parity suites touching 2-D chains, C1 bench line,
# launch list and one ncu --set full capture of the chain kernel
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_resident_smem.py tests/test_gpu_temporal.py tests/test_gpu_parity.py tests/test_gpu_integration.py -x -q > gpurun_out/rsm_suite.log 2>&1
echo "suite rc=$?"; tail -3 gpurun_out/rsm_suite.log
timeout 600 python bench.py --workload c1 > gpurun_out/c1_rsm.json 2> gpurun_out/c1_rsm.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_c1_rsm.csv python bench.py --workload c1 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/launches_c1_rsm.log 2>&1
echo "launches rc=$?"
bash scripts/ncu_kernel.sh c1 est_resident_smem c1_resident_smem
