cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for n in 2 4; do
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2957$n bench.py --gpus $n --steps 3 --warmup 3 > gpurun_out/bench_c4_n$n.log 2>&1; echo "n=$n rc=$?"; tail -1 gpurun_out/bench_c4_n$n.log | cut -c1-300
done
