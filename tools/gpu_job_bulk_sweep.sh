cd $GRAFT_REPO_ROOT
for cfg in 1024,16,3,1,0 2048,8,3,1,0 1024,8,6,1,1; do echo "parity $cfg: $(SDNN_BULK=$cfg timeout 120 python -m pytest tests/test_gpu_parity.py -x -q -k 'c1_full or ragged or hand or irregular or ka' 2>&1 | tail -1)"; done
for skew in 0 32 256 1024; do for cfg in 1024,32,1,1,0 1024,16,3,1,0; do
  SDNN_SKEW=$skew SDNN_BULK=$cfg timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 skew $skew', '$cfg', round(d['ms_per_step'],1), '%.3e'%d['value'], 'frac', round(d['roofline']['frac'],3))" 2>&1 | tail -1
done; done
