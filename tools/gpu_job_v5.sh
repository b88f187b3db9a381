cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/all_gpu_v5.log 2>&1; tail -1 gpurun_out/all_gpu_v5.log
for c in c4 c2; do timeout 900 python bench.py --config $c > gpurun_out/bench5_$c.json 2> gpurun_out/bench5_$c.err; tail -1 gpurun_out/bench5_$c.json | cut -c1-160; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass -s 200 -c 1 -o gpurun_out/prof_c4_pass_v5 python bench.py --oneshot --steps 1 --warmup 0 > /dev/null 2>&1; ls gpurun_out/*v5*
