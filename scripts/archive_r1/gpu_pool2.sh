cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/c5_scratch
EST_SCRATCH=$GRAFT_REPO_ROOT/gpurun_out/c5_scratch timeout 2400 python scripts/rescale_bench.py --n 32768 --iters 100 --workers 8 > gpurun_out/rescale_c5_32k.log 2>&1; echo "rescale32k rc=$?"; tail -1 gpurun_out/rescale_c5_32k.log | python -c "
import sys, json
d=json.loads(sys.stdin.read()); print(json.dumps(d['rescales'])); print(d['phase_glups'], d['bit_equal_to_unrescaled'])"
grep -h "restore:\|migrate " gpurun_out/c5_scratch/logs/gpu-worker-*.log | sort | cut -c1-250
rm -rf gpurun_out/c5_scratch
