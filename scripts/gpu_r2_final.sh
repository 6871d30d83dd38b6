# round-2 evidence run: full GPU suite, smoke, bench lines (C4 default + C1/C2/C3/lap16k, >= 20 steps), 2/4 ranks, C5 BASELINE shape
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
(nproc; lscpu | grep -E 'Model name|^CPU\(s\)'; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv) > gpurun_out/final/box_info.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?" | tee -a gpurun_out/final/smoke.log
timeout 900 python bench.py > gpurun_out/final/bench_c4.log 2>&1; tail -1 gpurun_out/final/bench_c4.log | cut -c1-200
for wl in c2 c3 lap16k; do timeout 900 python bench.py --workload $wl --steps 20 --warmup 5 > gpurun_out/final/bench_$wl.log 2>&1; tail -1 gpurun_out/final/bench_$wl.log | cut -c1-160; done
timeout 900 python bench.py --workload c1 > gpurun_out/final/bench_c1.log 2>&1; tail -1 gpurun_out/final/bench_c1.log | cut -c1-160
for n in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n bench.py --gpus $n --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/final/bench_c4_${n}r.log 2>&1; tail -1 gpurun_out/final/bench_c4_${n}r.log | cut -c1-160
done
rm -rf /tmp/est-r3-*
EST_WORKER_LOG=1 timeout 2400 python scripts/rescale3d_bench.py > gpurun_out/final/c5.json 2> gpurun_out/final/c5.err; echo "c5 rc=$?"; cut -c1-600 gpurun_out/final/c5.json
mkdir -p gpurun_out/final/c5logs; for d in /tmp/est-r3-*; do cp -r $d/logs gpurun_out/final/c5logs/$(basename $d) 2>/dev/null; done
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1500 -rfE > gpurun_out/final/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final/pytest_gpu.log
tail -12 gpurun_out/final/pytest_gpu.log
