cd $GRAFT_REPO_ROOT
bash tools/gpujob.sh r2q tests_fast bench:c4:--no-cpu-baseline,--e2e-steps,3 launches:c4 "full:c4:k_pass<.int.16, .int.1, .bool.0, .int.1>:40"
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "full_size_c4 or full_size_c3 or full_size_c2" > gpurun_out/r2q_full.log 2>&1; tail -1 gpurun_out/r2q_full.log
bash tools/gpujob.sh r2q_off env:SDNN_PASS_VT=0 bench:c4:--no-cpu-baseline,--e2e-steps,1
