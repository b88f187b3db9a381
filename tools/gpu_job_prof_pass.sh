cd $GRAFT_REPO_ROOT
timeout 400 python -m pytest tests/test_gpu_parity.py -x -q -k "fused" 2>&1 | tail -2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pass -s 200 -c 1 -o gpurun_out/prof_c4_pass python bench.py --oneshot --steps 1 --warmup 0 --fuse-rows 128 > gpurun_out/prof_c4_pass.log 2>&1; tail -2 gpurun_out/prof_c4_pass.log
