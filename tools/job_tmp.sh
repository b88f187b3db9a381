cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_flow_gpu.py -q -x > gpurun_out/r2g_flow.log 2>&1; tail -3 gpurun_out/r2g_flow.log
timeout 600 python tools/f1_launch_study.py c1 4 > gpurun_out/r2g_f1_c1.json 2>&1; tail -2 gpurun_out/r2g_f1_c1.json
timeout 900 python tools/f1_launch_study.py c2 4 > gpurun_out/r2g_f1_c2.json 2>&1; tail -2 gpurun_out/r2g_f1_c2.json
bash tools/gpujob.sh r2g bench:c4 bench:c3:--no-cpu-baseline,--e2e-steps,2 bench:c2:--no-cpu-baseline bench:c1:--no-cpu-baseline
bash tools/gpujob.sh r2g bench:c4:--net,rn-plain,--no-cpu-baseline,--e2e-steps,1:plain bench:c3:--net,rn-plain,--no-cpu-baseline,--e2e-steps,1:plain
