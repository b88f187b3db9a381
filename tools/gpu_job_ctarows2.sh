# cluster-size study after the unconditional chain fast path
cd $GRAFT_REPO_ROOT
for r in 128 512; do SDNN_PASS_CTA_ROWS=$r timeout 900 python -m pytest tests -m gpu -q -x -k "fused or c1_full or stream" > gpurun_out/cr2_tests_$r.log 2>&1; echo "rows=$r $(tail -1 gpurun_out/cr2_tests_$r.log)"; done
for r in 128 256 512; do
  SDNN_PASS_CTA_ROWS=$r timeout 900 python bench.py --config c4 --no-cpu-baseline --e2e-steps 1 > gpurun_out/cr2_bench_$r.json 2> gpurun_out/cr2_bench_$r.err
  echo "rows=$r $(tail -1 gpurun_out/cr2_bench_$r.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],1),'%.3e'%d['value'],d['roofline']['frac'],d['fuse'])")"; done
