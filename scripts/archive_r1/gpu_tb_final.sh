#!/bin/bash
# tb on by default (48x32, B only in the last chain): full GPU suite, smoke,
# bench lines, launch list + ncu capture of est_tb
cd "$(dirname "$0")/.."
bash scripts/gpu_full.sh
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_c4_tb.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/launches_c4_tb.log 2>&1
echo "launches rc=$?"
bash scripts/ncu_kernel.sh c4 est_tb c4_tb_48x32
bash scripts/ncu_kernel.sh c2 est_tb c2_tb_48x32
