set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fe_fem_rtc -s 2 -c 1 -f -o gpurun_out/prof_fem_rtc python tools/time_fused.py 1 fused > gpurun_out/ncu_fem_rtc.log 2>&1; echo ncu1=$?
timeout 600 python tools/time_fused.py 10 "fused,tables,meta=stages=4;ept=2;te=32,meta=stages=4;ept=1;te=32,meta=stages=2;ept=2;te=64,meta=stages=3;ept=1;te=64"
