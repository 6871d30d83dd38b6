# ncu --set full of every shipped dominant kernel at its bench geometry + launch list of the default bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash scripts/ncu_kernel.sh c4 est_tb r2b_c4_tb
bash scripts/ncu_kernel.sh c2 est_tb r2b_c2_tb
bash scripts/ncu_kernel.sh c3 est_stream r2b_c3_stream
bash scripts/ncu_kernel.sh c1 est_resident_smem r2b_c1_rsm
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2b_c4_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-check --no-seam > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
