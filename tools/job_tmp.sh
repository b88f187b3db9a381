cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash tools/gpujob.sh r3i tests smoke bench:c4 "bench:c3:--net,rw:rw"
