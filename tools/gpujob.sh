#!/bin/bash
# One GPU job script for gpurun (replaces the round-1 one-off gpu_job_*.sh).
#
#   gpurun --timeout 3000 -- 'bash tools/gpujob.sh TAG recipe [recipe ...]'
#
# Every recipe writes under gpurun_out/TAG_*; each is bounded by `timeout`.
#   tests        pytest -m gpu (all GPU tests, slow ones included)
#   tests_fast   pytest -m "gpu and not slow"
#   smoke        __graft_entry__.smoke()
#   bench:CFG[:ARGS]   bench.py --config CFG (ARGS: extra flags, ',' -> ' ')
#   launches:CFG[:ARGS[:SUFFIX]]  ncu launch list (gpu__time_duration, cold, serialised) of one inference
#   full:CFG:KREGEX[:SKIP]  ncu --set full of one launch of the kernels matching KREGEX
#   env:VAR=VAL  export for the following recipes
#   sanitize     compute-sanitizer memcheck / synccheck / racecheck on tools/sanitize_run.py
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=$1
shift
summ() {  # one-line summary of a bench JSON line
  tail -1 "$1" | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read())
except Exception as e:
    print('no json', e); sys.exit()
r=d.get('roofline') or {}
print(round(d['ms_per_step'],2),'ms','%.4e'%d['value'],'e2e %.4e'%((d.get('e2e') or {}).get('value') or 0),
      'frac',round(r.get('frac') or 0,3),'steps',(d.get('fuse') or {}).get('steps'))"
}
for R in "$@"; do
  IFS=: read -r K A B C <<< "$R"
  case $K in
    env) export "$A"; echo "env $A" ;;
    tests) timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_tests.log 2>&1
           echo "tests: $(tail -1 gpurun_out/${TAG}_tests.log)" ;;
    tests_fast) timeout 1500 python -m pytest tests -m "gpu and not slow" -q > gpurun_out/${TAG}_tests.log 2>&1
           echo "tests_fast: $(tail -1 gpurun_out/${TAG}_tests.log)" ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
           echo "smoke: $(tail -1 gpurun_out/${TAG}_smoke.log)" ;;
    bench) X=${B//,/ }; N=${TAG}_bench_${A}${C:+_$C}
           timeout 1200 python bench.py --config $A $X > gpurun_out/$N.json 2> gpurun_out/$N.err
           echo "bench $A $X: $(summ gpurun_out/$N.json)" ;;
    launches) X=${B//,/ }; N=${TAG}_launches_$A${C:+_$C}
              timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
                --log-file gpurun_out/$N.csv python bench.py --config $A $X --oneshot --steps 1 --warmup 0 \
                > /dev/null 2>&1
              python tools/ncu_summary.py launches gpurun_out/$N.csv 2>&1 | head -12 ;;
    full) timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
            -k "regex:$B" -s "${C:-60}" -c 1 -o gpurun_out/${TAG}_full_${A}_$(echo "$B" | tr -cd 'a-z0-9_') \
            python bench.py --config $A --oneshot --steps 1 --warmup 0 ${FULLARGS:-} > gpurun_out/${TAG}_full.log 2>&1
          REP=gpurun_out/${TAG}_full_${A}_$(echo "$B" | tr -cd 'a-z0-9_')
          # text summaries on the box (gpurun_out/ comes back only if < 64 MiB)
          ncu -i $REP.ncu-rep --page details > $REP.details.txt 2>/dev/null
          ncu -i $REP.ncu-rep --page raw --csv > $REP.raw.csv 2>/dev/null
          ncu -i $REP.ncu-rep --page source --csv --print-source sass > $REP.sass.csv 2>/dev/null
          [ "${KEEP_REP:-0}" = "1" ] || rm -f $REP.ncu-rep
          echo "full $A $B: $REP ($(grep -m1 Duration $REP.details.txt | tr -s ' '))" ;;
    sanitize) for tool in memcheck synccheck racecheck; do
                timeout 1500 compute-sanitizer --tool $tool python tools/sanitize_run.py \
                  > gpurun_out/${TAG}_sanitize_$tool.log 2>&1
                echo "$tool: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize_run ok' gpurun_out/${TAG}_sanitize_$tool.log | tr '\n' ' ')"
              done ;;
    *) echo "unknown recipe $R" ;;
  esac
done
