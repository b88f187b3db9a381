# usage: bash tools/gpu_job_abcfg.sh TAG CONFIG V1 V2 ... -- bench CONFIG for each library variant, interleaved x3
TAG=$1; CFG=$2; shift 2
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/all_gpu_$TAG.log 2>&1; tail -1 gpurun_out/all_gpu_$TAG.log
for rep in 1 2 3; do for v in "$@"; do
  if [ $v = main ]; then L=$PWD/paper_2004_10908_b200/libsdnn.so; else L=$PWD/paper_2004_10908_b200/libsdnn_$v.so; fi
  SDNN_LIB=$L timeout 900 python bench.py --config $CFG > gpurun_out/bench_${TAG}_${v}_$rep.json 2> gpurun_out/bench_${TAG}_${v}_$rep.err
  echo "$v rep$rep $(tail -1 gpurun_out/bench_${TAG}_${v}_$rep.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],3),d['roofline']['frac'])")"
done; done
