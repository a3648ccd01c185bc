set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "hex" > gpurun_out/t_hex.log 2>&1; echo pytest=$?; tail -3 gpurun_out/t_hex.log
timeout 900 python -m pytest tests/test_benched_parity.py -m gpu -x -q -p no:cacheprovider -k "C2 or hex" > gpurun_out/t_hexb.log 2>&1; echo pytestb=$?; tail -3 gpurun_out/t_hexb.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hex5 -c 1 -f -o gpurun_out/prof_hex5 python tools/run_variant.py C2 "" 1 > gpurun_out/ncu_hex5.log 2>&1; echo ncu=$?
