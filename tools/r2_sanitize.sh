timeout 300 python tools/sanitize_cases.py > gpurun_out/sanitize_plain.log 2>&1; echo plain=$?; tail -20 gpurun_out/sanitize_plain.log
bash tools/sanitize.sh memcheck,racecheck,synccheck,initcheck
