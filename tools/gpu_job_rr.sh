# RR (random 32-regular, no shared source lists): the general gather path beside RN
cd $GRAFT_REPO_ROOT
for c in c1 s1024x480 s4096x120 c2; do
  timeout 900 python bench.py --config $c --net rr --no-cpu-baseline --e2e-steps 1 > gpurun_out/rr_$c.json 2> gpurun_out/rr_$c.err
  echo "rr $c $(tail -1 gpurun_out/rr_$c.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],2),'%.3e'%d['value'],'e2e %.3e'%d['e2e']['value'],round(d['roofline']['frac'],3),d['fuse']['steps'],d['survivors']['categories'], d['roofline']['kernel'][:40])")"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rr_launches_c2.csv python bench.py --oneshot --config c2 --net rr --steps 1 --warmup 0 > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/rr_launches_c2.csv 2>&1 | head -8
