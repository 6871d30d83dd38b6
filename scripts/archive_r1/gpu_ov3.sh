cd $GRAFT_REPO_ROOT
for ov in 1 0; do for w in c3 c4; do
EST_OVERLAP=$ov timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2958$ov bench.py --gpus 2 --workload $w --steps 3 --warmup 3 > gpurun_out/b.log 2>&1
python -c "import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print('overlap=$ov $w n=2', round(d['value'],1))"
done; done
