# round 2 checkpoint run: full GPU suite, smoke, default bench, launch list, ncu of est_tb
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
(nproc; lscpu | grep -E 'Model name|^CPU\(s\)'; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv) > gpurun_out/box_info.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -rfE > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -30 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log; tail -4 gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c4.log 2>&1; tail -1 gpurun_out/bench_c4.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-check > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
bash scripts/ncu_kernel.sh c4 est_tb r2_c4_tb_full
