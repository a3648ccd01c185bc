# hex variant A/B: bitwise equality vs v2 and timing (C2 full size); HEXV="v=5 v=6"
set -x
for v in ${HEXV:-v=5}; do timeout 300 python tools/ab_compare.py C2 "" "$v" | sort | uniq -c | head -3; done
for r in 1 2; do timeout 300 python tools/run_variant.py C2 "" 3; for v in ${HEXV:-v=5}; do timeout 300 python tools/run_variant.py C2 "$v" 3; done; done
