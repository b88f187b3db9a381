set -x
cd $GRAFT_REPO_ROOT
nproc; lscpu | grep "Model name"; free -g | head -2
for t in memcheck racecheck synccheck; do timeout 600 compute-sanitizer --tool $t --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/sanitize_$t.log 2>&1; echo "$t rc=$?"; tail -3 gpurun_out/sanitize_$t.log; done
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -c 3000 gpurun_out/bench_c4.json
timeout 300 python bench.py --config c2 --no-cpu-baseline > gpurun_out/bench_c2.json 2>&1; tail -c 600 gpurun_out/bench_c2.json
timeout 300 python bench.py --config c2 --no-cpu-baseline --no-e2e --flags no_graph > gpurun_out/bench_c2_nograph.json 2>&1; tail -c 300 gpurun_out/bench_c2_nograph.json
timeout 300 python bench.py --config c1 --no-cpu-baseline --no-e2e > gpurun_out/bench_c1.json 2>&1; tail -c 300 gpurun_out/bench_c1.json
timeout 300 python bench.py --config c1 --no-cpu-baseline --no-e2e --flags no_graph > gpurun_out/bench_c1_nograph.json 2>&1; tail -c 300 gpurun_out/bench_c1_nograph.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_bulk.csv python bench.py --oneshot --steps 1 --warmup 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_layer_bulk -s 300 -c 1 -o gpurun_out/prof_c4_bulk python bench.py --oneshot --steps 1 --warmup 0 > gpurun_out/prof_c4_bulk.log 2>&1; tail -2 gpurun_out/prof_c4_bulk.log
