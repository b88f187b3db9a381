# 512-row single-CTA passes (T = 32..512 tiles) + 4-layer cluster passes: tests, C4/C3 bench, launch list
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -k "fused or c1_full or stream or signed or smoke" > gpurun_out/t32_tests.log 2>&1; tail -3 gpurun_out/t32_tests.log
for cap in 512 2048 128; do timeout 900 python bench.py --config c4 --fuse-rows $cap --no-cpu-baseline --e2e-steps 1 > gpurun_out/t32_bench_$cap.json 2> gpurun_out/t32_bench_$cap.err
  echo "cap=$cap $(tail -1 gpurun_out/t32_bench_$cap.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],1),'%.3e'%d['value'],d['roofline']['frac'],d['fuse'])")"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_t32.csv python bench.py --oneshot --steps 1 --warmup 0 > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/launches_c4_t32.csv 2>&1 | head -20
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/t32_all.log 2>&1; tail -2 gpurun_out/t32_all.log
