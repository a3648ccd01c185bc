# e2e (fe_plan_execute_host) per config under host-pipeline overrides
for envs in "" "FE_PIPE_MIN_MB=1 FE_PIPE_CHUNKS=2" "FE_PIPE_MIN_MB=1 FE_PIPE_CHUNKS=4" "FE_PIPE_MIN_MB=1 FE_PIPE_CHUNKS=8" "FE_PIPE_CHUNKS=16"; do
  env $envs timeout 600 python bench.py --configs ${CFGS:-C1,C4-f64,C4-f32,C5} --steps 3 --warmup 3 --no-extras --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$envs', {k:(round(v['ms'],3), round(v['pcie_frac'],2)) for k,v in d['e2e']['per_config'].items()})"
done
