# usage: bash scripts/ncu_kernel.sh <workload> <kernel regex> <out name> [extra env assignments...]
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
W=$1; K=$2; O=$3; shift 3
env "$@" timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/$O \
  python bench.py --workload $W --steps 1 --warmup 1 --no-cpu-baseline --no-check > gpurun_out/$O.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/$O.log
