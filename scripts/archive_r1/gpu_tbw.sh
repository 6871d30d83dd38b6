cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_temporal.py -q -p no:cacheprovider --timeout 300 -k "tb" > gpurun_out/pytest_tbw.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_tbw.log
run() { env EST_TB=1 "$@" timeout 600 python bench.py --workload c4 --steps 4 --warmup 2 --no-cpu-baseline > gpurun_out/c4w.log 2>&1; python -c "import json; d=json.loads(open('gpurun_out/c4w.log').read().strip().splitlines()[-1]); print('$*', round(d['value'],1), round(d['roofline']['frac'],3), round(d['roofline']['kernel_ms'],3), d['roofline']['kernel'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1; }
run EST_TB_MINB=1
run EST_TB_MINB=2
run EST_TB_R=3 EST_TB_MINB=1
run EST_TB_R=3 EST_TB_MINB=2
run EST_TB_R=2 EST_TB_MINB=2
run EST_TB_WY=2 EST_TB_MINB=2
run EST_TB_WX=4 EST_TB_WY=2 EST_TB_MINB=1
run EST_TB_PREFETCH=4 EST_TB_MINB=1
