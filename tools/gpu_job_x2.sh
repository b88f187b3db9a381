cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/all_gpu_x2.log 2>&1; tail -1 gpurun_out/all_gpu_x2.log
for rep in 1 2; do for v in main nox2; do for cap in -1 128; do
  if [ $v = main ]; then L=$PWD/paper_2004_10908_b200/libsdnn.so; else L=$PWD/paper_2004_10908_b200/libsdnn_$v.so; fi
  SDNN_LIB=$L timeout 900 python bench.py --config c4 --fuse-rows $cap --no-cpu-baseline > gpurun_out/bench_x2_${v}_${cap}_$rep.json 2> gpurun_out/bench_x2_${v}_${cap}_$rep.err
  echo "$v cap=$cap rep$rep $(tail -1 gpurun_out/bench_x2_${v}_${cap}_$rep.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],1),d['roofline']['frac'])")"
done; done; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_x2.csv python bench.py --oneshot --steps 1 --warmup 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass -s 150 -c 1 -o gpurun_out/prof_c4_x2 python bench.py --oneshot --steps 1 --warmup 0 > /dev/null 2>&1; ls gpurun_out/*x2*rep
