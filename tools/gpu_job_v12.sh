# v12 (position-blocked activations default): all GPU tests, smoke, sanitizers, C1-C4 bench, launch list, ncu full of the top pass kernels
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/v12_gpu_tests.log 2>&1; tail -1 gpurun_out/v12_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v12_smoke.log 2>&1; tail -1 gpurun_out/v12_smoke.log
for t in memcheck synccheck racecheck; do timeout 600 compute-sanitizer --tool $t --print-limit 3 python tools/sanitize_run.py > gpurun_out/v12_san_$t.log 2>&1; echo "$t: $(grep -h 'SUMMARY\|sanitize_run ok' gpurun_out/v12_san_$t.log | tr '\n' ' ')"; done
for c in c1 c2 c3 c4; do timeout 900 python bench.py --config $c > gpurun_out/v12_bench_$c.json 2> gpurun_out/v12_bench_$c.err; echo "$c $(tail -1 gpurun_out/v12_bench_$c.json | cut -c1-200)"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/v12_launches_c4.csv python bench.py --oneshot --steps 1 --warmup 0 > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/v12_launches_c4.csv 2>&1 | head -12
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_pass<.int.32, .int.1, .bool.0>" -s 60 -c 1 -o gpurun_out/v12_prof_p32c1 python bench.py --oneshot --steps 1 --warmup 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_pass<.int.32, .int.2, .bool.1>" -s 60 -c 1 -o gpurun_out/v12_prof_p32c2 python bench.py --oneshot --steps 1 --warmup 0 > /dev/null 2>&1
ls gpurun_out/v12*.ncu-rep
