# cost-weighted pass cover (SDNN_PLAN=cost) vs greedy on C4 / C3, fused parity under it
cd $GRAFT_REPO_ROOT
SDNN_PLAN=cost timeout 900 python -m pytest tests -m gpu -q -x -k "fused or blocked or ragged or c1_full or full_size_c2" > gpurun_out/pl_tests.log 2>&1; tail -1 gpurun_out/pl_tests.log
for c in c4 c3; do for p in cost greedy; do
  SDNN_PLAN=$p timeout 900 python bench.py --config $c --no-cpu-baseline --e2e-steps 1 > gpurun_out/pl_${c}_$p.json 2> gpurun_out/pl_${c}_$p.err
  echo "$c $p $(tail -1 gpurun_out/pl_${c}_$p.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],1),'%.3e'%d['value'],round(d['roofline']['frac'],3),d['fuse']['steps'],round(d['load_seconds'],1))")"; done; done
