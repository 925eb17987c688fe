#!/bin/bash
# Development A/B on the GPU box with tight timeouts: smoke, the forward parity
# tests, then device/e2e timings of library variants (base = product library).
# Usage (under gpurun): bash scripts/quick_ab.sh [--tests] base VARIANT ...
mkdir -p gpurun_out
if [ "$1" = --tests ]; then
  shift
  timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
  timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_keyed_layer0.py -x -q 2>&1 | tail -1
  timeout 300 python -m pytest tests/test_gpu_scale.py -x -q 2>&1 | tail -1
fi
for v in "$@"; do
  lib=paper_2511_18297_b200/libgroot_b200.so
  [ "$v" != base ] && lib=paper_2511_18297_b200/libgroot_b200_$v.so
  GROOT_LIB=$PWD/$lib timeout 150 python bench.py --no-cpu-baseline --no-side --steps 10 --e2e-steps 3 > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  python -c "
import json,sys
try:
    d=json.load(open('gpurun_out/ab_$v.json')); k=d['kernels']
    c=d.get('clocks',{})
    print('$v', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],2), {x:round(v['ms_per_launch'],3) for x,v in k.items() if 'sage' in x or 'l0' in x}, c.get('sm_mhz'), c.get('power_w_median'), c.get('power_cap_samples'), c.get('samples'))
except Exception as e:
    print('$v failed', e)" 
done
