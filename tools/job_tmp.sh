cd $GRAFT_REPO_ROOT
bash tools/gpujob.sh r2f tests_fast bench:c4:--no-cpu-baseline,--e2e-steps,1 launches:c4
bash tools/gpujob.sh r2f_nb1 env:SDNN_PASS_NB=1 bench:c4:--no-cpu-baseline,--e2e-steps,1
bash tools/gpujob.sh r2f_rw bench:c3:--net,rw,--no-cpu-baseline,--e2e-steps,1 bench:c4:--net,rw,--no-cpu-baseline,--e2e-steps,1
