cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none -k regex:est_stream -s 5 -c 1 -o gpurun_out/lap16k python scripts/lap_sweep.py > gpurun_out/lap16k.log 2>&1; echo rc=$?
