cd $GRAFT_REPO_ROOT
for pad in 1 0; do echo "pad $pad: $(SDNN_RES_PAD=$pad timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k 'resident or c1_full' 2>&1 | tail -1)"; done
for pad in 1 0; do for c in c1 c2; do SDNN_RES_PAD=$pad timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pad $pad $c', round(d['ms_per_step'],3), '%.3e'%d['value'])"; done; done
timeout 300 compute-sanitizer --tool racecheck --print-limit 5 --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/racecheck.log 2>&1; grep -E "Race reported|RACECHECK SUMMARY" gpurun_out/racecheck.log | head -4
