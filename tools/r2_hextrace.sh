set -x
timeout 300 python tools/hex_trace.py C2 3
for r in 1 2; do timeout 300 python tools/run_variant.py C2 "" 3; done
