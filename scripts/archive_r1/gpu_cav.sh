cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 300 -k "cavity or random or golden_case_single" > gpurun_out/pytest_cav.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_cav.log
timeout 900 python scripts/paper_bench.py > gpurun_out/paper_bench.json 2>gpurun_out/paper_bench.err; echo rc=$?; python -c "
import json; d=json.load(open('gpurun_out/paper_bench.json'))
for k,v in d.items(): print(k, {kk: round(vv,3) if isinstance(vv,float) else vv for kk,vv in v.items()})"
