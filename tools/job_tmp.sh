cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash tools/gpujob.sh r2x tests smoke bench:c4 bench:c3 bench:c2 bench:c1 launches:c4
