# position-blocked activations (SDNN_YBLOCK=1): GPU tests under it, C4/C3 A/B
cd $GRAFT_REPO_ROOT
SDNN_YBLOCK=1 timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/yb_tests.log 2>&1; tail -1 gpurun_out/yb_tests.log
for c in c4 c3; do for y in 1; do
  SDNN_YBLOCK=$y timeout 900 python bench.py --config $c --no-cpu-baseline --e2e-steps 1 > gpurun_out/yb_bench_${c}_$y.json 2> gpurun_out/yb_bench_${c}_$y.err
  echo "$c yblk=$y $(tail -1 gpurun_out/yb_bench_${c}_$y.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],1),'%.3e'%d['value'],d['roofline']['frac'],d['fuse'])")"; done; done
SDNN_YBLOCK=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/yb_launches_c4.csv python bench.py --oneshot --steps 1 --warmup 0 > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/yb_launches_c4.csv 2>&1 | head -8
