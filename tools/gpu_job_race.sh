cd $GRAFT_REPO_ROOT
for cfg in 512,32,3,1,0 1024,16,3,1,0 1024,32,1,1,0; do SDNN_BULK=$cfg timeout 300 compute-sanitizer --tool racecheck --print-limit 1 python tools/sanitize_run.py > gpurun_out/rc_$cfg.log 2>&1; done
grep -H "RACECHECK SUMMARY" gpurun_out/rc_*.log
