# where the 2-rank (one GPU) C4 efficiency goes: halo windows / overlap on-off
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-seam --no-check > gpurun_out/b1.log 2>&1; tail -1 gpurun_out/b1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('1 rank', round(d['value'],1), round(d['roofline']['kernel_ms'],3), d['clocks']['sm_mhz'])"
for cfg in "EST_HALO_WINDOWS=1" "EST_HALO_WINDOWS=0" "EST_OVERLAP=0" "EST_PDL=0"; do
env $cfg timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b2.log 2>&1; tail -1 gpurun_out/b2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg 2 ranks', round(d['value'],1), round(d['roofline']['kernel_ms'],3), round(d['roofline']['kernel_ms_isolated'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/b2.log
done
