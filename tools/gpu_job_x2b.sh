cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/all_gpu_x2b.log 2>&1; tail -1 gpurun_out/all_gpu_x2b.log
for rep in 1 2; do for v in main nox2 v2; do for cap in -1 128; do
  L=$PWD/paper_2004_10908_b200/libsdnn.so; E=""
  [ $v = nox2 ] && L=$PWD/paper_2004_10908_b200/libsdnn_nox2.so
  [ $v = v2 ] && E="SDNN_PASS_V=2"
  env $E SDNN_LIB=$L timeout 900 python bench.py --config c4 --fuse-rows $cap --no-cpu-baseline > gpurun_out/bench_x2b_${v}_${cap}_$rep.json 2> gpurun_out/bench_x2b_${v}_${cap}_$rep.err
  echo "$v cap=$cap rep$rep $(tail -1 gpurun_out/bench_x2b_${v}_${cap}_$rep.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],1),d['roofline']['frac'])")"
done; done; done
