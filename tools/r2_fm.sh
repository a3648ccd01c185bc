set -x
timeout 600 python tools/time_fused.py 10 "fused,tables"
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo pytest=$?; tail -5 gpurun_out/gputest.log
