cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/all_gpu_x2c.log 2>&1; tail -1 gpurun_out/all_gpu_x2c.log
SDNN_PASS_V=2 timeout 600 python -m pytest tests -m "gpu and not slow" -q -x -k "fused or c1_full or stream or signed" > gpurun_out/v2_tests.log 2>&1; tail -1 gpurun_out/v2_tests.log
for rep in 1 2; do for x in 0 1; do SDNN_PASS_X2=$x timeout 900 python bench.py --config c4 --no-cpu-baseline > gpurun_out/bench_x2c_${x}_$rep.json 2> gpurun_out/bench_x2c_${x}_$rep.err
  echo "x2_c1=$x rep$rep $(tail -1 gpurun_out/bench_x2c_${x}_$rep.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],1),d['roofline']['frac'])")"; done; done
for c in c1 c2 c3 c4; do timeout 900 python bench.py --config $c > gpurun_out/bench_r01v9_$c.json 2> gpurun_out/bench_r01v9_$c.err; echo "$c $(tail -1 gpurun_out/bench_r01v9_$c.json | cut -c1-200)"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_v9.csv python bench.py --oneshot --steps 1 --warmup 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass -s 150 -c 1 -o gpurun_out/prof_c4_v9 python bench.py --oneshot --steps 1 --warmup 0 > /dev/null 2>&1; ls gpurun_out/*v9*
