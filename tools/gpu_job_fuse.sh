cd $GRAFT_REPO_ROOT
timeout 400 python -m pytest tests/test_gpu_parity.py -x -q -k "fused" > gpurun_out/fuse_tests.log 2>&1; tail -1 gpurun_out/fuse_tests.log
for fr in 128 0; do timeout 600 python bench.py --no-cpu-baseline --no-e2e --fuse-rows $fr > gpurun_out/fuse_c4_$fr.log 2>&1; tail -1 gpurun_out/fuse_c4_$fr.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 fuse', $fr, round(d['ms_per_step'],1), '%.3e'%d['value'], 'frac', round(d['roofline']['frac'],3), d['fuse'])"; done
for fr in 128 0; do timeout 300 python bench.py --config c3 --no-cpu-baseline --no-e2e --fuse-rows $fr 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 fuse', $fr, round(d['ms_per_step'],1), '%.3e'%d['value'], d['fuse'])"; done
