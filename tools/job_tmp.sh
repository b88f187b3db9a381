cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/e2e_probe.py c2 > gpurun_out/r3d_probe_c2.log 2>&1; tail -6 gpurun_out/r3d_probe_c2.log
SDNN_PASS_WIDE=1 timeout 600 python tools/e2e_probe.py c2 > gpurun_out/r3d_probe_c2_w1.log 2>&1; tail -6 gpurun_out/r3d_probe_c2_w1.log
bash tools/gpujob.sh r3d bench:c2 bench:c2::rep "bench:c4:--net,rn-plain:plain" "bench:c3:--net,rn-plain:plain" "bench:c4:--net,rw:rw" "bench:c3:--net,rw:rw"
