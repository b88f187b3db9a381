cd $GRAFT_REPO_ROOT
SDNN_PASS=1,16,4,8192,1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "fused" 2>&1 | tail -1
SDNN_PASS=2,8,2,8192,2 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "fused" 2>&1 | tail -1
for cfg in 1,8,5,8192,1 1,8,2,8192,2 1,16,4,8192,1 1,16,2,8192,2 2,8,2,16384,1 2,4,2,8192,2 2,8,2,8192,2 1,4,1,8192,4; do
  SDNN_PASS=$cfg timeout 600 python bench.py --no-cpu-baseline --no-e2e --fuse-rows 128 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4', '$cfg', round(d['ms_per_step'],1), '%.3e'%d['value'], 'frac', round(d['roofline']['frac'],3), d['fuse']['steps'])" 2>&1 | tail -1
done
