#!/bin/bash
# Round profiling recipe (run under gpurun, 1 GPU). Writes into gpurun_out/.
#   bash profiles/collect.sh [configs]
CFG=${1:-C1,C3,C5}
set -x
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --configs $CFG --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:fem_grad -s 2 -c 1 -f -o gpurun_out/prof_fem \
  python bench.py --configs C5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gett -s 1 -c 1 -f -o gpurun_out/prof_gett \
  python bench.py --configs C3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out
