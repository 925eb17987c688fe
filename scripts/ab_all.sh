#!/bin/bash
# A/B of env knobs: forward per-kernel ms (bench.py) and the standalone SpMM.
for cfg in "$@"; do
  env $cfg timeout 600 python bench.py --no-cpu-baseline --steps 5 --e2e-steps 1 > gpurun_out/ab.json 2>&1
  python -c "
import json,sys; d=json.load(open('gpurun_out/ab.json')); k=d['kernels']
print('$cfg', round(d['ms_per_step'],2), {x:round(v['ms_per_launch'],2) for x,v in k.items() if 'tc' in x or 'layer0' in x}, 'spmm', round(d['spmm']['ms'],2))" || tail -2 gpurun_out/ab.json
done
