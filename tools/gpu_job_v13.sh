# v13 (1024-row single-CTA passes, T = 16, one-layer passes in blocked plans): tests, smoke, C1-C4, launch list, ncu full
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/v13_gpu_tests.log 2>&1; tail -1 gpurun_out/v13_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v13_smoke.log 2>&1; tail -1 gpurun_out/v13_smoke.log
for c in c4 c3 c2 c1; do timeout 900 python bench.py --config $c > gpurun_out/v13_bench_$c.json 2> gpurun_out/v13_bench_$c.err
  echo "$c $(tail -1 gpurun_out/v13_bench_$c.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],2),'%.3e'%d['value'],'e2e %.3e'%d['e2e']['value'],round(d['roofline']['frac'],3),d['fuse'])")"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/v13_launches_c4.csv python bench.py --oneshot --steps 1 --warmup 0 > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/v13_launches_c4.csv 2>&1 | head -9
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_pass<.int.16, .int.1, .bool.0>" -s 60 -c 1 -o gpurun_out/v13_prof_p16 python bench.py --oneshot --steps 1 --warmup 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_pass<.int.32, .int.1, .bool.0>" -s 60 -c 1 -o gpurun_out/v13_prof_p32 python bench.py --oneshot --steps 1 --warmup 0 > /dev/null 2>&1
ls gpurun_out/v13*.ncu-rep
