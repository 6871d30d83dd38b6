# est_tc diagnosis: sanitizer on the fp32 V=2 rotation, ncu of est_tc (C3 wave, paper-shape Laplace), e2e probe with the new hash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
EST_TC_VEC=8 timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_temporal2d.py -x -q -p no:cacheprovider -k "64-6-1" > gpurun_out/tc_sanitize.log 2>&1; grep -m20 -E "=====|Invalid|Error|error|passed|failed" gpurun_out/tc_sanitize.log
bash scripts/ncu_kernel.sh c3 est_tc r2_c3_tc_full
bash scripts/ncu_kernel.sh lap16k est_tc r2_lap16k_tc_full
timeout 600 python scripts/e2e_probe.py c4 12 > gpurun_out/e2e_probe_c4.log 2>&1; tail -13 gpurun_out/e2e_probe_c4.log
