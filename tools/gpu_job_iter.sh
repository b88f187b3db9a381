# usage: bash tools/gpu_job_iter.sh TAG  -- GPU tests, C4 + C2 bench, ncu full capture of one k_pass launch
TAG=${1:-x}
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/all_gpu_$TAG.log 2>&1; tail -3 gpurun_out/all_gpu_$TAG.log
for c in c4 c2; do timeout 900 python bench.py --config $c > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err; tail -1 gpurun_out/bench_${TAG}_$c.json | cut -c1-160; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass -s 200 -c 1 -o gpurun_out/prof_c4_pass_$TAG python bench.py --oneshot --steps 1 --warmup 0 > /dev/null 2>&1; ls gpurun_out/*$TAG*
