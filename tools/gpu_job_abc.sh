# usage: bash tools/gpu_job_abc.sh TAG V1 V2 ...  -- C4 bench for each prebuilt library variant
# (paper_2004_10908_b200/libsdnn_<V>.so; "main" = libsdnn.so), same box, interleaved twice
TAG=$1; shift
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/all_gpu_$TAG.log 2>&1; tail -1 gpurun_out/all_gpu_$TAG.log
for rep in 1 2; do for v in "$@"; do
  if [ $v = main ]; then L=$PWD/paper_2004_10908_b200/libsdnn.so; else L=$PWD/paper_2004_10908_b200/libsdnn_$v.so; fi
  SDNN_LIB=$L timeout 900 python bench.py --config c4 > gpurun_out/bench_${TAG}_${v}_$rep.json 2> gpurun_out/bench_${TAG}_${v}_$rep.err
  echo "$v rep$rep $(tail -1 gpurun_out/bench_${TAG}_${v}_$rep.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],1),d['roofline']['frac'])")"
done; done
