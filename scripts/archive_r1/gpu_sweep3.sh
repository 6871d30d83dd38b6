cd $GRAFT_REPO_ROOT
timeout 900 python scripts/stream_sweep.py --sustained > gpurun_out/sweep3.jsonl 2> gpurun_out/sweep3.err; cat gpurun_out/sweep3.jsonl; tail -3 gpurun_out/sweep3.err
timeout 900 python scripts/stream_sweep.py > gpurun_out/sweep3_burst.jsonl 2>&1; cat gpurun_out/sweep3_burst.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:est_stream --csv --log-file gpurun_out/sweep3_ncu.csv python scripts/stream_sweep.py --ncu > gpurun_out/sweep3_ncu.jsonl 2>&1
EST_STREAM_WS=1 EST_STREAM_ZREG=1 timeout 600 python scripts/debug_stream.py rand3d > gpurun_out/debug_ws.log 2>&1; tail -2 gpurun_out/debug_ws.log
EST_STREAM_WS=1 EST_STREAM_ZREG=1 timeout 600 python scripts/debug_stream.py heat3d >> gpurun_out/debug_ws.log 2>&1; tail -2 gpurun_out/debug_ws.log
EST_STREAM_WS=1 EST_STREAM_ZREG=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "heat3d or rand3d or random_programs" > gpurun_out/pytest_ws.log 2>&1; tail -2 gpurun_out/pytest_ws.log
