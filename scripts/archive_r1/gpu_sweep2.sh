cd $GRAFT_REPO_ROOT
timeout 900 python scripts/stream_sweep.py > gpurun_out/sweep2.jsonl 2> gpurun_out/sweep2.err; cat gpurun_out/sweep2.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:est_stream --csv --log-file gpurun_out/sweep2_ncu.csv python scripts/stream_sweep.py --ncu > gpurun_out/sweep2_ncu.jsonl 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_default.log 2>&1; tail -1 gpurun_out/bench_default.log
