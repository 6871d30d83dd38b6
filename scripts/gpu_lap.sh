cd $GRAFT_REPO_ROOT
for cfg in "128 48 4 2" "128 32 4 2" "128 32 4 3" "128 24 4 3" "128 16 4 3" "128 24 6 2" "128 40 4 2" "64 32 4 3"; do
  set -- $cfg
  EST_STREAM2D_BX=$1 EST_STREAM2D_BY=$2 EST_STREAM2D_TY=$3 EST_STREAM2D_PREFETCH=$4 timeout 300 python scripts/lap_sweep.py 2>&1 | tail -1
done
