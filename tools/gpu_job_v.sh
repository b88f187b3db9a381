# pass kernel shapes: GPU tests (both shapes), C4 bench V x cap, launch list + ncu of top pass kernel
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/all_gpu_pv.log 2>&1; tail -1 gpurun_out/all_gpu_pv.log
SDNN_PASS_V=4 timeout 600 python -m pytest tests -m "gpu and not slow" -q -x -k "fused or c1_full or stream or signed" > gpurun_out/v4_tests.log 2>&1; tail -1 gpurun_out/v4_tests.log
for V in 2 4; do for cap in -1 128; do SDNN_PASS_V=$V timeout 900 python bench.py --config c4 --fuse-rows $cap > gpurun_out/bench_pv_${V}_$cap.json 2> gpurun_out/bench_pv_${V}_$cap.err
  echo "V=$V cap=$cap $(tail -1 gpurun_out/bench_pv_${V}_$cap.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],1),'%.3e'%d['value'],d['roofline']['frac'],d['fuse']['steps'])")"; done; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_pv.csv python bench.py --oneshot --steps 1 --warmup 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass -s 150 -c 1 -o gpurun_out/prof_c4_pv python bench.py --oneshot --steps 1 --warmup 0 > /dev/null 2>&1; ls gpurun_out/*pv*
