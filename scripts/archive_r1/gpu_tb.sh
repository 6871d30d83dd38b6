cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export EST_TB=1
for cfg in "64 16 2 4 0 0 128" "64 16 2 6 0 0 128" "64 16 2 8 0 0 128" "64 16 2 4 0 1 128" "64 16 2 6 0 1 128" "64 16 2 6 0 1 256" "64 16 2 6 0 0 256" "64 22 4 6 0 1 128" "128 8 2 6 0 1 128"; do
  set -- $cfg
  EST_TB_BX=$1 EST_TB_BY=$2 EST_TB_RPT=$3 EST_TB_PREFETCH=$4 EST_TB_MINB=$5 EST_TB_PERSISTENT=$6 EST_TB_ZCHUNK=$7 timeout 600 python bench.py --workload c4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/c4tb.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/c4tb.log').read().strip().splitlines()[-1]); print('c4 tb $cfg', round(d['value'],1), round(d['roofline']['frac'],3), round(d['roofline']['kernel_ms'],3), d['roofline']['kernel'], d['clocks']['sm_mhz'])" 2>&1 | tail -1
done
