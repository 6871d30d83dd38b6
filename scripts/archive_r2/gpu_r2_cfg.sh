cd $GRAFT_REPO_ROOT
(nproc; free -g; lscpu | head -20; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv) > gpurun_out/box_info.txt 2>&1
timeout 1700 python -m pytest tests/test_gpu_bench_configs.py -q -s -p no:cacheprovider --timeout 1200 -rA > gpurun_out/bench_cfg.log 2>&1; echo "rc=$?" >> gpurun_out/bench_cfg.log
tail -15 gpurun_out/bench_cfg.log
