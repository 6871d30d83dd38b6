cd $GRAFT_REPO_ROOT
set -x
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
for sk in point stream; do
  timeout 600 python bench.py --steps 5 --warmup 3 --skeleton $sk --no-cpu-baseline > gpurun_out/bench_$sk.log 2>&1; tail -2 gpurun_out/bench_$sk.log
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 120 --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:est_stream -s 3 -c 1 -o gpurun_out/prof_c4_stream python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_stream.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:est_node -s 3 -c 1 -o gpurun_out/prof_c4_point python bench.py --steps 1 --warmup 1 --no-cpu-baseline --skeleton point > gpurun_out/ncu_point.log 2>&1
ls -la gpurun_out
