# usage: bash tools/gpu_job_ab.sh TAG VAR  -- GPU tests, then C4 bench with VAR=0 and VAR=1, ncu of k_pass (VAR default)
TAG=${1:-x}; VAR=${2:-SDNN_PASS_GATHER}
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/all_gpu_$TAG.log 2>&1; tail -3 gpurun_out/all_gpu_$TAG.log
for v in 0 1; do env $VAR=$v timeout 900 python bench.py --config c4 > gpurun_out/bench_${TAG}_${v}.json 2> gpurun_out/bench_${TAG}_${v}.err; echo "$VAR=$v"; tail -1 gpurun_out/bench_${TAG}_${v}.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['ms_per_step'],d['value'],d['roofline']['frac'])"; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass -s 200 -c 1 -o gpurun_out/prof_c4_pass_$TAG python bench.py --oneshot --steps 1 --warmup 0 > /dev/null 2>&1; ls gpurun_out/*$TAG*
