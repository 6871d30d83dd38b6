cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/launches_c4.log 2>&1; echo "launches rc=$?"
bash scripts/ncu_kernel.sh c4 est_stream c4_stream_ws2
bash scripts/ncu_kernel.sh c3 est_stream c3_stream_ws2
bash scripts/ncu_kernel.sh c2 est_stream c2_stream_ws2
