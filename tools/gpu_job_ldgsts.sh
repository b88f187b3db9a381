# LDGSTS row loads for tiles <= 128 positions: parity subset, C4 bench (512 / 128 rows per CTA), launch list
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -k "fused or c1_full or stream or smoke" > gpurun_out/lg_tests.log 2>&1; tail -1 gpurun_out/lg_tests.log
for r in 512 128; do
  SDNN_PASS_CTA_ROWS=$r timeout 900 python bench.py --config c4 --no-cpu-baseline --e2e-steps 1 > gpurun_out/lg_bench_$r.json 2> gpurun_out/lg_bench_$r.err
  echo "rows=$r $(tail -1 gpurun_out/lg_bench_$r.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],1),'%.3e'%d['value'],d['roofline']['frac'],d['fuse'])")"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_lg.csv python bench.py --oneshot --steps 1 --warmup 0 > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/launches_c4_lg.csv 2>&1 | head -7
