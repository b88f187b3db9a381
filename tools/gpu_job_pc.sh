# cost-cover penalty A/B on C4 (SDNN_PLAN_COST="big,small")
cd $GRAFT_REPO_ROOT
for pc in "0.3,0" "0.2,0" "0.45,0" "0.3,0.1"; do
  SDNN_PLAN_COST=$pc timeout 900 python bench.py --config c4 --no-cpu-baseline --no-e2e > gpurun_out/pc_$pc.json 2> gpurun_out/pc_$pc.err
  echo "pc=$pc $(tail -1 gpurun_out/pc_$pc.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],1),'%.3e'%d['value'],d['fuse']['steps'])")"; done
