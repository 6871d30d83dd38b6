cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_temporal.py -q -p no:cacheprovider --timeout 300 > gpurun_out/pytest_chains.log 2>&1; echo "chains rc=$?"; tail -3 gpurun_out/pytest_chains.log
for r in 1 0; do
EST_RESIDENT=$r timeout 600 python bench.py --workload c1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1.log 2>&1; echo "c1 rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/bench_c1.log').read().strip().splitlines()[-1]); print('c1 resident=$r', round(d['value'],1), d['ms_per_step'], round(d['roofline']['frac'],3), d['roofline']['kernel'], round(d['roofline']['kernel_ms'],4), 'e2e', round(d['e2e']['value'],1), d['gpu_launches'])"
done
