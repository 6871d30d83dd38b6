cd $GRAFT_REPO_ROOT
timeout 600 python scripts/debug_stream.py rand3d > gpurun_out/debug_stream.log 2>&1; echo "rc=$?" >> gpurun_out/debug_stream.log
tail -5 gpurun_out/debug_stream.log
if grep -q FAULT gpurun_out/debug_stream.log; then
  timeout 600 compute-sanitizer --tool memcheck python scripts/debug_stream.py rand3d_000 > gpurun_out/sanitizer.log 2>&1; grep -m 20 -E "Invalid|Error|error|=========" gpurun_out/sanitizer.log | head -40
fi
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_stream2.log 2>&1; tail -1 gpurun_out/bench_stream2.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:est_stream -s 3 -c 1 -o gpurun_out/prof_c4_stream2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
