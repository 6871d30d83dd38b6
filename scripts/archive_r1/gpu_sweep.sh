cd $GRAFT_REPO_ROOT
timeout 900 python scripts/stream_sweep.py > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err; cat gpurun_out/sweep.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -k regex:est_stream --csv --log-file gpurun_out/sweep_ncu.csv python scripts/stream_sweep.py --ncu > gpurun_out/sweep_ncu.jsonl 2>&1
tail -3 gpurun_out/sweep_ncu.jsonl
timeout 1200 python -m pytest tests/test_gpu_ipc.py tests/test_gpu_integration.py -x -q -p no:cacheprovider > gpurun_out/pytest_ipc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ipc.log; tail -5 gpurun_out/pytest_ipc.log
