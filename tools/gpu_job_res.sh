# resident tail vs fused passes only on C1 / C2 / C3
cd $GRAFT_REPO_ROOT
for c in c1 c2; do for f in "" no_resident; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --e2e-steps 1 --flags "$f" > gpurun_out/rs_bench_${c}_$f.json 2> gpurun_out/rs_bench_${c}_$f.err
  echo "$c flags=$f $(tail -1 gpurun_out/rs_bench_${c}_$f.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],3),'%.3e'%d['value'],d['fuse'])")"; done; done
