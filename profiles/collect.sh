#!/bin/bash
# Round profiling recipe (run under gpurun, 1 GPU). Writes into gpurun_out/.
#   bash profiles/collect.sh [configs]
# 1) the launch list (per-kernel durations, cold cache, serialised) of a short bench run;
# 2) one `ncu --set full` capture of each config's dominant kernel.
CFG=${1:-C1,C2,C3,C4-f64,C4-f32,C5}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --configs $CFG --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-extras > gpurun_out/ncu_launches.log 2>&1
for spec in "fem_grad C5" "gett C3" "tt_kernel C4-f64" "tt_kernel C4-f32" "hex5 C2" "fem_grad C1"; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$1 -s 2 -c 1 -f -o gpurun_out/prof_${1}_$2 \
    python bench.py --configs $2 --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ncu_${1}_$2.log 2>&1
done
ls -la gpurun_out
