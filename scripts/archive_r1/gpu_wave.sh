cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_temporal.py -q -p no:cacheprovider --timeout 120 -x -k "wave" > gpurun_out/pytest_wave.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_wave.log
run() { env "$@" timeout 300 python bench.py --workload $W --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/cv.log 2>&1; python -c "import json; d=json.loads(open('gpurun_out/cv.log').read().strip().splitlines()[-1]); print('$W $*', round(d['value'],1), round(d['roofline']['frac'],3), round(d['roofline']['kernel_ms'],3), d['roofline']['kernel'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1; }
W=c2
run EST_WAVE=1 EST_WAVE_ZBLOCK=8
run EST_WAVE=1 EST_WAVE_ZBLOCK=16
run EST_WAVE=1 EST_WAVE_ZBLOCK=16 EST_WAVE_LEAD=3
run EST_WAVE=1 EST_WAVE_ZBLOCK=32
W=c4
run EST_WAVE=1 EST_WAVE_ZBLOCK=4
run EST_WAVE=1 EST_WAVE_ZBLOCK=8
run EST_WAVE=1 EST_WAVE_ZBLOCK=16
EST_WAVE=1 EST_WAVE_ZBLOCK=16 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:est_wave -s 3 -c 1 python bench.py --workload c2 --steps 1 --warmup 1 --no-cpu-baseline 2>&1 | grep -E "dram__|gpu__time|lts__" | head -6
