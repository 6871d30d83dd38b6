# C5 stage split with per-buffer arenas (EST_POOL_GROW=1) vs the default 4x arenas
cd $GRAFT_REPO_ROOT
for g in 1 4; do
rm -rf /tmp/est-r3-*; mkdir -p gpurun_out/c5logs_g$g
EST_POOL_GROW=$g EST_WORKER_LOG=1 timeout 1500 python scripts/rescale3d_bench.py --iters 200 --batches 2 > gpurun_out/c5probe_g$g.json 2> gpurun_out/c5probe_g$g.err; echo "grow $g rc=$?"
python -c "import json; d=json.load(open('gpurun_out/c5probe_g$g.json')); print(json.dumps(d['rescales']), d['bit_equal_to_unrescaled'], d['glups'])"
for d in /tmp/est-r3-*; do cp -r $d/logs gpurun_out/c5logs_g$g/$(basename $d) 2>/dev/null; done
grep -h "migrate" gpurun_out/c5logs_g$g/*/gpu-*-err.log | cut -c1-250 | head -16
done
