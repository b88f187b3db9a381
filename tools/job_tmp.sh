cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=$GRAFT_REPO_ROOT/paper_2004_10908_b200
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "knob or c2 or c4 or c1" > gpurun_out/r3a_t.log 2>&1; tail -1 gpurun_out/r3a_t.log
bash tools/gpujob.sh r3a bench:c4::regs env:SDNN_LIB=$L/libsdnn_r0.so bench:c4::shfl env:SDNN_LIB=$L/libsdnn.so bench:c4::regs2 "full:c4:k_pass_t32<.int.4:60"
