set -x
timeout 900 python -m pytest tests/test_epilogue.py -m gpu -x -q -p no:cacheprovider > gpurun_out/t_fused.log 2>&1; echo pytest=$?; tail -5 gpurun_out/t_fused.log
timeout 600 python tools/time_fused.py 10 "fused,epi,meta=stages=4;ept=2;te=32,meta=stages=4;ept=1;te=32;dsmem=1,meta=stages=4;ept=1;te=32,meta=stages=3;ept=1;te=16;dsmem=1,meta=stages=6;ept=1;te=16;dsmem=1,meta=stages=4;ept=2;te=68"
