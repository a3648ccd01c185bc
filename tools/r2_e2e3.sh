for envs in "" "FE_NO_ROWPIPE=1" "" "FE_COPY_ROWS=64"; do
  env $envs timeout 900 python bench.py --configs C1,C2,C4-f64 --steps 3 --warmup 3 --no-extras --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('[$envs]', d['e2e']['pcie'], {k:(round(v['ms'],3), round(v['pcie_frac'],2)) for k,v in d['e2e']['per_config'].items()})"
done
