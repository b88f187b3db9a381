# liveness-word spread: fused parity subset + C4 bench
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -k "fused or ragged or c1_full or smoke" > gpurun_out/lv_tests.log 2>&1; tail -1 gpurun_out/lv_tests.log
timeout 900 python bench.py --config c4 --no-cpu-baseline --e2e-steps 1 > gpurun_out/lv_bench.json 2> gpurun_out/lv_bench.err
tail -1 gpurun_out/lv_bench.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],1),'%.3e'%d['value'],d['roofline']['frac'],d['fuse'])"
