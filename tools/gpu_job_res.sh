cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "resident or c1_full" 2>&1 | tail -1
for c in c1 c2; do timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],3), '%.3e'%d['value'])"; done
timeout 900 ncu --set full --clock-control none -k regex:k_resident -c 1 -o gpurun_out/prof_c2_res2 python bench.py --oneshot --config c2 --steps 1 --warmup 0 > /dev/null 2>&1; echo profiled
