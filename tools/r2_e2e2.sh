for envs in "FE_COPY_ROWS=64" "FE_COPY_ROWS=0" "FE_COPY_ROWS=64" "FE_COPY_ROWS=0"; do
  env $envs timeout 900 python bench.py --steps 3 --warmup 3 --no-extras --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$envs', round(d['e2e']['value'],1), {k:(round(v['ms'],3), round(v['pcie_frac'],2)) for k,v in d['e2e']['per_config'].items()})"
done
