cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 300 -k "large_2d or wave2d or laplace or random or golden_case_single" > gpurun_out/pytest_2d.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_2d.log
for w in c1 c3; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$w.log 2>&1; echo "$w rc=$?"
  python -c "import json; d=json.loads(open('gpurun_out/bench_$w.log').read().strip().splitlines()[-1]); print('$w', round(d['value'],1), round(d['roofline']['frac'],3), round(d['roofline']['kernel_ms'],4), d['e2e']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1
done
