# blocked layout: component cap 512 / 2048 vs the default 1024 on C4
cd $GRAFT_REPO_ROOT
for cap in 512 2048; do
  timeout 900 python bench.py --config c4 --fuse-rows $cap --no-cpu-baseline --e2e-steps 1 > gpurun_out/caps2_$cap.json 2> gpurun_out/caps2_$cap.err
  echo "cap=$cap $(tail -1 gpurun_out/caps2_$cap.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],1),'%.3e'%d['value'],round(d['roofline']['frac'],3),d['fuse'])")"; done
