cd $GRAFT_REPO_ROOT
timeout 400 python -m pytest tests/test_gpu_parity.py -x -q -k "fused or c1" 2>&1 | tail -2
for fr in 256 128 64 0; do timeout 600 python bench.py --no-cpu-baseline --no-e2e --fuse-rows $fr 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 fuse', $fr, round(d['ms_per_step'],1), '%.3e'%d['value'], 'hbm-frac', round(d['roofline']['frac'],3), d['fuse'])"; done
for fr in 256 128 0; do timeout 300 python bench.py --config c2 --no-cpu-baseline --no-e2e --fuse-rows $fr 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2 fuse', $fr, round(d['ms_per_step'],2), '%.3e'%d['value'], 'hbm-frac', round(d['roofline']['frac'],3), d['fuse'])"; done
