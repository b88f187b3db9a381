# segmented float4 pass kernel: parity subset, C4 bench caps 512/2048/128, X2 A/B, launch list
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -k "fused or c1_full or stream or signed or smoke" > gpurun_out/seg_tests.log 2>&1; tail -3 gpurun_out/seg_tests.log
for cfg in "512 0" "512 1" "2048 0" "128 0"; do set -- $cfg
  SDNN_PASS_X2=$2 timeout 900 python bench.py --config c4 --fuse-rows $1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/seg_bench_$1_$2.json 2> gpurun_out/seg_bench_$1_$2.err
  echo "cap=$1 x2=$2 $(tail -1 gpurun_out/seg_bench_$1_$2.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],1),'%.3e'%d['value'],d['roofline']['frac'],d['fuse'])")"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_seg.csv python bench.py --oneshot --steps 1 --warmup 0 > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/launches_c4_seg.csv 2>&1 | head -14
