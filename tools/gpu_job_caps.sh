# component caps 512 / 1024 / 2048 with LDGSTS small tiles; ncu full of k_pass<32,1,0>
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -k "fused or c1_full" > gpurun_out/caps_tests.log 2>&1; tail -1 gpurun_out/caps_tests.log
for cap in 512 1024 2048; do
  timeout 900 python bench.py --config c4 --fuse-rows $cap --no-cpu-baseline --e2e-steps 1 > gpurun_out/caps_bench_$cap.json 2> gpurun_out/caps_bench_$cap.err
  echo "cap=$cap $(tail -1 gpurun_out/caps_bench_$cap.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],1),'%.3e'%d['value'],d['roofline']['frac'],d['fuse'])")"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_caps2048.csv python bench.py --oneshot --steps 1 --warmup 0 --fuse-rows 2048 > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/launches_c4_caps2048.csv 2>&1 | head -8
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_pass<.int.32, .int.1, .bool.0>" -s 100 -c 1 -o gpurun_out/prof_t32c python bench.py --oneshot --steps 1 --warmup 0 > gpurun_out/prof_t32c.log 2>&1
