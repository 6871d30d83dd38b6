cd $GRAFT_REPO_ROOT
timeout 900 python scripts/stream_sweep.py --sustained > gpurun_out/sweep4.jsonl 2> gpurun_out/sweep4.err; cat gpurun_out/sweep4.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:est_stream --csv --log-file gpurun_out/sweep4_ncu.csv python scripts/stream_sweep.py --ncu > gpurun_out/sweep4_ncu.jsonl 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r1.log 2>&1; tail -1 gpurun_out/bench_r1.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 30 -c 300 --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:est_stream -s 5 -c 1 -o gpurun_out/prof_c4_final python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 900 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 --workload c2 > gpurun_out/bench_2proc.log 2>&1; tail -2 gpurun_out/bench_2proc.log
timeout 600 python bench.py --workload c1 --steps 10 --warmup 3 > gpurun_out/bench_c1.log 2>&1; tail -1 gpurun_out/bench_c1.log
