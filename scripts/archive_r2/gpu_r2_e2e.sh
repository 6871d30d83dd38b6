cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for wl in c4 lap16k; do timeout 600 python scripts/e2e_probe.py $wl 16 > gpurun_out/e2e_probe_$wl.log 2>&1; cat gpurun_out/e2e_probe_$wl.log | tail -18; done
