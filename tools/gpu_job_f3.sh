# f3: GPU tests, then C4 bench resident vs weight streaming (same box)
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/all_gpu_f3.log 2>&1; tail -1 gpurun_out/all_gpu_f3.log
for S in 0 2 4; do timeout 900 python bench.py --config c4 --stream-slots $S > gpurun_out/bench_f3_s$S.json 2> gpurun_out/bench_f3_s$S.err
  echo "slots=$S $(tail -1 gpurun_out/bench_f3_s$S.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],1),'%.3e'%d['value'],'e2e %.3e'%d['e2e']['value'],d.get('weight_streaming'))")"; done
