# re-entry check: all GPU tests, smoke, default bench (C4)
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r1b_smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r1b_gpu_tests.log 2>&1; tail -2 gpurun_out/r1b_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1b_smoke.log 2>&1; tail -1 gpurun_out/r1b_smoke.log
timeout 900 python bench.py > gpurun_out/r1b_bench.json 2> gpurun_out/r1b_bench.err; tail -1 gpurun_out/r1b_bench.json | cut -c1-300
