cd $GRAFT_REPO_ROOT
run() { env "$@" timeout 600 python bench.py --workload c4 --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/c4x.log 2>&1; python -c "import json; d=json.loads(open('gpurun_out/c4x.log').read().strip().splitlines()[-1]); print('$*', round(d['value'],1), round(d['roofline']['frac'],3), round(d['roofline']['kernel_ms'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1; }
run EST_STREAM_BX=128 EST_STREAM_BY=16 EST_STREAM_TY=4 EST_STREAM_PREFETCH=3
run EST_STREAM_BX=128 EST_STREAM_BY=24 EST_STREAM_TY=3 EST_STREAM_PREFETCH=2
run EST_STREAM_BX=128 EST_STREAM_BY=24 EST_STREAM_TY=4 EST_STREAM_PREFETCH=2
run EST_STREAM_BX=128 EST_STREAM_BY=32 EST_STREAM_TY=4 EST_STREAM_PREFETCH=2
run EST_STREAM_BX=128 EST_STREAM_BY=20 EST_STREAM_TY=4 EST_STREAM_PREFETCH=2
run EST_STREAM_BX=64 EST_STREAM_BY=32 EST_STREAM_TY=4 EST_STREAM_PREFETCH=3
run EST_STREAM_BX=128 EST_STREAM_BY=16 EST_STREAM_TY=4 EST_STREAM_PREFETCH=3
