# C5 stage breakdown: worker logs (migrate / restore splits) of one 8->4->8 run
cd $GRAFT_REPO_ROOT
rm -rf /tmp/est-r3-*; mkdir -p gpurun_out/c5logs
EST_WORKER_LOG=1 timeout 1500 python scripts/rescale3d_bench.py --iters 200 --batches 2 > gpurun_out/c5probe.json 2> gpurun_out/c5probe.err; echo "rc=$?"
python -c "import json; d=json.load(open('gpurun_out/c5probe.json')); print(json.dumps(d['rescales']), d['bit_equal_to_unrescaled'])"
for d in /tmp/est-r3-*; do cp -r $d/logs gpurun_out/c5logs/$(basename $d) 2>/dev/null; done
grep -h "migrate\|restore" gpurun_out/c5logs/*/gpu-*-err.log | cut -c1-400 | head -60
