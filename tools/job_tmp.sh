cd $GRAFT_REPO_ROOT
bash tools/gpujob.sh r2d tests_fast
for pf in 0 1 2; do bash tools/gpujob.sh r2d_pf$pf env:SDNN_PASS_PF=$pf bench:c4:--no-cpu-baseline,--e2e-steps,1; done
bash tools/gpujob.sh r2d env:SDNN_PASS_PF=1 launches:c4
bash tools/gpujob.sh r2d_rw bench:c3:--net,rw,--no-cpu-baseline,--e2e-steps,1 bench:c4:--net,rw,--no-cpu-baseline,--e2e-steps,1
