# parallel pinned staging: e2e on C2 / C4, host-path GPU tests
cd $GRAFT_REPO_ROOT
nproc
timeout 900 python -m pytest tests -m gpu -q -x -k "c1_full or hand or signed or abi" > gpurun_out/e2_tests.log 2>&1; tail -1 gpurun_out/e2_tests.log
for c in c2 c4; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/e2_bench_$c.json 2> gpurun_out/e2_bench_$c.err
  echo "$c $(tail -1 gpurun_out/e2_bench_$c.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],2),'%.3e'%d['value'],'e2e', round(d['e2e']['ms_per_step'],2), '%.3e'%d['e2e']['value'])")"; done
