cd $GRAFT_REPO_ROOT
bash tools/gpujob.sh r2n tests_fast bench:c4:--no-cpu-baseline,--e2e-steps,1 launches:c4 bench:c2:--no-cpu-baseline,--e2e-steps,1
bash tools/gpujob.sh r2n_x2 env:SDNN_PASS_X2=16 bench:c4:--no-cpu-baseline,--e2e-steps,1
