cd $GRAFT_REPO_ROOT
timeout 900 python tools/e2e_probe.py c4 2>&1 | tail -6
SDNN_IN_CHUNK_MB=4096 timeout 900 python tools/e2e_probe.py c4 2>&1 | tail -6
