cd $GRAFT_REPO_ROOT
for cfg in "128 48 2 2" "128 64 2 2" "128 40 2 2" "128 48 1 2" "128 56 2 2" "128 48 2 3" "128 32 1 2"; do
  set -- $cfg
  EST_STREAM2D_BX=$1 EST_STREAM2D_BY=$2 EST_STREAM2D_TY=$3 EST_STREAM2D_PREFETCH=$4 timeout 300 python scripts/lap_sweep.py 2>&1 | tail -1
done
for cfg in "128 48 4 2" "128 48 2 2" "128 64 2 2"; do
  set -- $cfg
  EST_STREAM2D_BX=$1 EST_STREAM2D_BY=$2 EST_STREAM2D_TY=$3 EST_STREAM2D_PREFETCH=$4 timeout 600 python bench.py --workload c3 --steps 4 --warmup 2 --no-cpu-baseline > gpurun_out/c3s.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/c3s.log').read().strip().splitlines()[-1]); print('c3 $cfg', round(d['value'],1), round(d['roofline']['frac'],3))"
done
