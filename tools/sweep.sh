# BASELINE configs[4]: width/depth sweep 1024-65536 neurons x 120-1920 layers, 60,000 inputs, one B200
cd $GRAFT_REPO_ROOT
out=gpurun_out/sweep.jsonl; : > $out
for n in 1024 4096 16384 65536; do for l in 120 480 1920; do
  timeout 900 python bench.py --config s${n}x${l} --no-cpu-baseline --e2e-steps 1 2> gpurun_out/sweep_${n}_${l}.err | tail -1 >> $out
done; done
python - <<'PY'
import json
print(f"{'N':>6} {'L':>5} {'ms/step':>9} {'edges/s':>10} {'e2e':>10} {'HBM frac':>8} {'steps':>6} {'cats':>6}")
for line in open("gpurun_out/sweep.jsonl"):
    try: d = json.loads(line)
    except Exception: continue
    c = d["config"]
    print(f"{c['neurons']:>6} {c['layers']:>5} {d['ms_per_step']:>9.2f} {d['value']:>10.3e} {d['e2e']['value']:>10.3e} "
          f"{d['roofline']['frac']:>8.3f} {d['fuse']['steps']:>6} {d['survivors']['categories']:>6}")
PY
