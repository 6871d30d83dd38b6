cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_temporal.py -q -x -p no:cacheprovider --timeout 600 > gpurun_out/tb_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tb_tests.log; tail -5 gpurun_out/tb_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log; tail -4 gpurun_out/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; tail -1 gpurun_out/bench_c4.log
timeout 1500 python -m pytest tests/test_gpu_bench_configs.py -q -x -p no:cacheprovider --timeout 1200 -k c4 > gpurun_out/bench_cfg.log 2>&1; echo "rc=$?" >> gpurun_out/bench_cfg.log; tail -5 gpurun_out/bench_cfg.log
