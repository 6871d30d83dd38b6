cd $GRAFT_REPO_ROOT
for h in 0 1 0 1; do
EST_STREAM_STHINT=$h timeout 600 python bench.py --workload c4 --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/c4h.log 2>&1; python -c "import json; d=json.loads(open('gpurun_out/c4h.log').read().strip().splitlines()[-1]); print('sthint=$h', round(d['value'],1), round(d['roofline']['frac'],3), round(d['roofline']['kernel_ms'],3), d['clocks']['sm_mhz'])"
done
EST_STREAM_STHINT=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:est_stream -s 3 -c 1 python bench.py --workload c4 --steps 1 --warmup 1 --no-cpu-baseline 2>&1 | grep -E "dram__|gpu__time" | head -3
