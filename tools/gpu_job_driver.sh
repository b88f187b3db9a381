# the driver's round-end commands, as it runs them
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/drv_build.log 2>&1; echo "build rc=$?"
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/drv_tests.log 2>&1; tail -1 gpurun_out/drv_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/drv_smoke.log 2>&1; tail -1 gpurun_out/drv_smoke.log
timeout 900 python bench.py --impl reference > gpurun_out/drv_ref.json 2> gpurun_out/drv_ref.err; tail -1 gpurun_out/drv_ref.json | cut -c1-200
timeout 900 python bench.py > gpurun_out/drv_bench.json 2> gpurun_out/drv_bench.err; tail -1 gpurun_out/drv_bench.json | cut -c1-200
