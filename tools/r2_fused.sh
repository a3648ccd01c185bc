for c in fem_mma fem_grad fem_rtc; do
  timeout 600 compute-sanitizer --tool initcheck --print-limit 3 python tools/sanitize_cases.py $c > gpurun_out/initcheck_$c.log 2>&1; echo "$c rc=$?"; grep -E "ERROR SUMMARY|cases ok" gpurun_out/initcheck_$c.log
done
timeout 900 python -m pytest tests/test_epilogue.py -m gpu -x -q -p no:cacheprovider > gpurun_out/t_fused.log 2>&1; echo pytest=$?; tail -5 gpurun_out/t_fused.log
timeout 600 python tools/time_fused.py 10 "fused,epi,meta=stages=4;ept=2;te=32,meta=stages=4;ept=1;te=32,meta=stages=4;ept=2;te=68,meta=stages=2;ept=2;te=64"
