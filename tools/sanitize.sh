#!/bin/bash
# compute-sanitizer over every kernel family (tools/sanitize_cases.py), under gpurun:
#   bash tools/sanitize.sh [tools] [cases]   -> gpurun_out/sanitize_<tool>.log
TOOLS=${1:-memcheck,racecheck,synccheck,initcheck}
CASES=${2:-}
for t in ${TOOLS//,/ }; do
  extra=""
  [ "$t" = "memcheck" ] && extra="--leak-check no"
  [ "$t" = "racecheck" ] && extra="--racecheck-report all"
  timeout 1500 compute-sanitizer --tool $t $extra --target-processes all --print-limit 50 \
    python tools/sanitize_cases.py $CASES > gpurun_out/sanitize_$t.log 2>&1
  echo "$t rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|all cases ok|Error|error" gpurun_out/sanitize_$t.log | head -8
done
