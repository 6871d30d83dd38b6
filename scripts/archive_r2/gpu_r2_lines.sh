# bench lines with >= 20 clock samples (long timed regions) + ncu of the shipped est_tc
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/lines
timeout 900 python bench.py --workload c2 --steps 80 --warmup 5 > gpurun_out/lines/bench_c2.log 2>&1; tail -1 gpurun_out/lines/bench_c2.log | cut -c1-120
timeout 900 python bench.py --workload c3 --steps 50 --warmup 5 > gpurun_out/lines/bench_c3.log 2>&1; tail -1 gpurun_out/lines/bench_c3.log | cut -c1-120
timeout 900 python bench.py --workload lap16k --steps 50 --warmup 5 > gpurun_out/lines/bench_lap16k.log 2>&1; tail -1 gpurun_out/lines/bench_lap16k.log | cut -c1-120
timeout 900 python bench.py --workload c1 --steps 8000 --warmup 5 > gpurun_out/lines/bench_c1.log 2>&1; tail -1 gpurun_out/lines/bench_c1.log | cut -c1-120
bash scripts/ncu_kernel.sh lap16k est_tc r2b_lap16k_tc
