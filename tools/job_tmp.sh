cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "knob or c2 or c3 or c4 or c1" > gpurun_out/r2q_t.log 2>&1; tail -1 gpurun_out/r2q_t.log
bash tools/gpujob.sh r2q bench:c4 env:SDNN_PASS_T32_S=2 bench:c4::s2 env:SDNN_PASS_T32=2 bench:c4::m2s2 env:SDNN_PASS_T32_S=1 bench:c4::m2s1 env:SDNN_PASS_T32=0 bench:c4::m0
