cd $GRAFT_REPO_ROOT
bash tools/gpujob.sh r2o sanitize tests
