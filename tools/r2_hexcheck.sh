set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "hex" > gpurun_out/t_hex.log 2>&1; echo pytest=$?; tail -3 gpurun_out/t_hex.log
timeout 900 python -m pytest tests/test_benched_parity.py -m gpu -x -q -p no:cacheprovider -k "C2 or hex" > gpurun_out/t_hexb.log 2>&1; echo pytestb=$?; tail -3 gpurun_out/t_hexb.log
for tool in memcheck racecheck synccheck; do timeout 900 compute-sanitizer --tool $tool --print-limit 5 python tools/sanitize_cases.py hex5 > gpurun_out/san_hex5_$tool.log 2>&1; echo $tool=$?; grep -E "SUMMARY|Error|hex" gpurun_out/san_hex5_$tool.log | head -3; done
for r in 1 2; do timeout 300 python tools/run_variant.py C2 "" 3; timeout 300 python tools/run_variant.py C2 "v=6" 3; done
