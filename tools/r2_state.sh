set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo pytest=$?; tail -5 gpurun_out/gputest.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?; tail -c 3000 gpurun_out/bench.json
timeout 600 python tools/time_fused.py 10 "fused,epi" > gpurun_out/fused.log 2>&1; echo fused=$?; tail -20 gpurun_out/fused.log
