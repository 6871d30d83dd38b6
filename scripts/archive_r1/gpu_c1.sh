cd $GRAFT_REPO_ROOT
for cfg in "64 16 2 2 1" "64 16 2 3 1" "64 16 1 2 1" "64 32 2 2 1" "32 16 2 2 1" "64 24 2 2 1" "32 32 2 2 1" "64 8 2 2 1"; do set -- $cfg
EST_STREAM2DS_BX=$1 EST_STREAM2DS_BY=$2 EST_STREAM2DS_TY=$3 EST_STREAM2DS_PREFETCH=$4 EST_STREAM2DS_PERSISTENT=$5 timeout 600 python bench.py --workload c1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c1.log 2>&1
python -c "import json; d=json.loads(open('gpurun_out/c1.log').read().strip().splitlines()[-1]); print('c1 $cfg', round(d['value'],1), round(d['ms_per_step'],4))"
done
