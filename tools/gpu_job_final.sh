# round-end check: every GPU test, smoke, default bench (C4), X2 A/B on C4
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/fin_gpu_tests.log 2>&1; tail -1 gpurun_out/fin_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; tail -1 gpurun_out/fin_smoke.log
timeout 900 python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err; tail -1 gpurun_out/fin_bench.json | cut -c1-250
SDNN_PASS_X2=1 timeout 900 python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/fin_bench_x2.json 2> gpurun_out/fin_bench_x2.err
tail -1 gpurun_out/fin_bench_x2.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print('x2', round(d['ms_per_step'],1),'%.3e'%d['value'])"
