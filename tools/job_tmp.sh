cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash tools/gpujob.sh r3t tests smoke
