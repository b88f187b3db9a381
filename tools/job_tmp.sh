cd $GRAFT_REPO_ROOT
bash tools/gpujob.sh r2j tests_fast bench:c4:--no-cpu-baseline,--e2e-steps,1 bench:c2:--no-cpu-baseline,--e2e-steps,1 bench:c3:--no-cpu-baseline,--e2e-steps,1 launches:c4
