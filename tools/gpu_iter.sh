#!/bin/bash
# One GPU iteration on a kernel: parity tests (pytest -k), timing and an ncu
# capture of one kernel.  bash tools/gpu_iter.sh <pytest -k expr> <config> <meta> <kernel regex> [tag]
K=$1; CFG=$2; META=$3; KER=$4; TAG=${5:-iter}
timeout 400 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "$K" > gpurun_out/t_$TAG.log 2>&1; echo pytest=$?; tail -3 gpurun_out/t_$TAG.log
timeout 200 python tools/run_variant.py $CFG "$META" 4
if [ -n "$KER" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$KER -c 1 -f -o gpurun_out/prof_$TAG python tools/run_variant.py $CFG "$META" 1 > gpurun_out/ncu_$TAG.log 2>&1; echo ncu=$?
fi
