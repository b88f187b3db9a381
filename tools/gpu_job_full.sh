cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m "gpu and not slow" -q > gpurun_out/all_gpu.log 2>&1; tail -1 gpurun_out/all_gpu.log
for c in c1 c2 c3 c4; do timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -1 gpurun_out/bench_$c.json | cut -c1-120; done
timeout 600 compute-sanitizer --tool memcheck python tools/sanitize_run.py > gpurun_out/san_mem.log 2>&1; tail -1 gpurun_out/san_mem.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_v4.csv python bench.py --oneshot --steps 1 --warmup 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass -s 200 -c 1 -o gpurun_out/prof_c4_pass_v4 python bench.py --oneshot --steps 1 --warmup 0 > /dev/null 2>&1; ls gpurun_out/*.ncu-rep
