cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/c5_scratch
timeout 1500 python -m pytest tests/test_gpu_ipc.py tests/test_gpu_integration.py tests/test_gpu_bench.py -q -p no:cacheprovider --timeout 600 > gpurun_out/pytest_pool.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_pool.log
timeout 1500 python scripts/rescale3d_bench.py --n 1024 --iters 100 > gpurun_out/r3d_c5.log 2>&1; echo c5-3d rc=$?; tail -1 gpurun_out/r3d_c5.log | python -c "
import sys, json
d=json.loads(sys.stdin.read()); print(d['redistribute_ms'], d['stage_ms_max_over_ranks'], d['glups'], d['bit_equal_to_unrescaled'])"
EST_SCRATCH=$GRAFT_REPO_ROOT/gpurun_out/c5_scratch timeout 2400 python scripts/rescale_bench.py --n 32768 --iters 100 --workers 8 > gpurun_out/rescale_c5_32k.log 2>&1; echo "rescale32k rc=$?"; tail -1 gpurun_out/rescale_c5_32k.log | python -c "
import sys, json
d=json.loads(sys.stdin.read()); print(json.dumps(d['rescales'])); print(d['phase_glups'], d['bit_equal_to_unrescaled'])"
grep -h "restore:\|migrate " gpurun_out/c5_scratch/logs/gpu-worker-*.log | sort | head -12
rm -rf gpurun_out/c5_scratch
