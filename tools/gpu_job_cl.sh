# cluster passes: GPU tests, C4 bench default (cap 512) vs cap 128, ncu of one k_pass_cl launch
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m "gpu and not slow" -q -x -k "fused or c1_full or stream or signed" > gpurun_out/cl_tests.log 2>&1; tail -3 gpurun_out/cl_tests.log
timeout 1200 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/all_gpu_cl.log 2>&1; tail -1 gpurun_out/all_gpu_cl.log
for cap in -1 128; do timeout 900 python bench.py --config c4 --fuse-rows $cap > gpurun_out/bench_cl_$cap.json 2> gpurun_out/bench_cl_$cap.err
  echo "cap=$cap $(tail -1 gpurun_out/bench_cl_$cap.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],1),'%.3e'%d['value'],d['roofline']['frac'],d['fuse'])")"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_cl.csv python bench.py --oneshot --steps 1 --warmup 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass_cl -s 150 -c 1 -o gpurun_out/prof_c4_cl python bench.py --oneshot --steps 1 --warmup 0 > /dev/null 2>&1; ls gpurun_out/*cl*
