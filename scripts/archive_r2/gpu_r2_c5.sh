# round 2: acceptance criteria 5/6 detail, C5 3-D rescale, C2/C3/C1 bench lines, tb sweep
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export PYTHONPATH=$GRAFT_REPO_ROOT/tests:$GRAFT_REPO_ROOT:$PYTHONPATH
(cd baseline/_ref/ref_tests && timeout 900 python -m pytest -p refsuite_plugin -q -p no:cacheprovider -s -k "criterion_5 or criterion_6" test_acceptance.py > $GRAFT_REPO_ROOT/gpurun_out/acc56.log 2>&1; echo "rc=$?" >> $GRAFT_REPO_ROOT/gpurun_out/acc56.log)
tail -5 gpurun_out/acc56.log
timeout 1500 python scripts/rescale3d_bench.py > gpurun_out/c5_3d.json 2> gpurun_out/c5_3d.err; echo "c5 rc=$?"; tail -c 1500 gpurun_out/c5_3d.json
for wl in c2 c3 c1; do
  timeout 900 python bench.py --workload $wl --steps 40 --warmup 5 > gpurun_out/bench_$wl.log 2>&1; tail -1 gpurun_out/bench_$wl.log | cut -c1-300
done
: > gpurun_out/sweep.log
for cfg in "EST_TB_L2PROMO=2" "EST_TB_L2PROMO=0" "EST_TB_PREFETCH=4" "EST_TB_PREFETCH=6" "EST_TB_RPT=4" "EST_TB_BY=16" "EST_TB_ZCHUNK=1024" "EST_TB_ZCHUNK=96"; do
  echo "== $cfg" >> gpurun_out/sweep.log
  env $cfg timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-check > gpurun_out/sweep_one.log 2>&1
  tail -1 gpurun_out/sweep_one.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['kernel_ms'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> gpurun_out/sweep.log 2>&1 || tail -3 gpurun_out/sweep_one.log >> gpurun_out/sweep.log
done
cat gpurun_out/sweep.log
