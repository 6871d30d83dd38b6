cd $GRAFT_REPO_ROOT
for pdl in 1 0; do
EST_PDL=$pdl timeout 600 python bench.py --workload c1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c1.log 2>&1
python -c "import json; d=json.loads(open('gpurun_out/c1.log').read().strip().splitlines()[-1]); print('c1 pdl=$pdl', round(d['value'],1), round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value'],1))"
done
EST_PDL=1 timeout 600 python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c4.log 2>&1; python -c "import json; d=json.loads(open('gpurun_out/c4.log').read().strip().splitlines()[-1]); print('c4 pdl=1', round(d['value'],1), round(d['roofline']['frac'],3))"
timeout 600 python scripts/paper_bench.py 2>/dev/null | grep -A2 "cavity_8192sq_f64\"" | head -3
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
