cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "c1_full or edge or ragged or pipelined or device_api" > gpurun_out/r2t_t.log 2>&1; tail -1 gpurun_out/r2t_t.log
for mb in 64 256 4096; do echo "chunk $mb MB"; SDNN_IN_CHUNK_MB=$mb timeout 900 python tools/e2e_probe.py c4 2>&1 | grep -E "K=8|sync, SDNN"; done
