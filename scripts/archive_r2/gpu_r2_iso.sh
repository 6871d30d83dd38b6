cd $GRAFT_REPO_ROOT
rm -rf /tmp/est-r3-*; mkdir -p gpurun_out/iso
timeout 2400 python -m pytest tests/test_gpu_rescale3d.py tests/test_gpu_integration.py -q -p no:cacheprovider --timeout 1500 -rfE > gpurun_out/iso/tests.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/iso/tests.log
for k in 1 2; do
rm -rf /tmp/est-r3-*
EST_WORKER_LOG=1 timeout 1500 python scripts/rescale3d_bench.py --iters 200 --batches 2 > gpurun_out/iso/c5probe$k.json 2> gpurun_out/iso/c5probe$k.err; echo "rc=$?"
python -c "import json; d=json.load(open('gpurun_out/iso/c5probe$k.json')); print(json.dumps(d['rescales']), d['bit_equal_to_unrescaled'], d['glups'])"
done
mkdir -p gpurun_out/iso/logs; for d in /tmp/est-r3-*; do cp -r $d/logs gpurun_out/iso/logs/$(basename $d) 2>/dev/null; done
grep -h "migrate" gpurun_out/iso/logs/*/gpu-*-err.log | cut -c1-250 | head -20
