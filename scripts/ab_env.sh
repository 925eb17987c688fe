#!/bin/bash
# GPU A/B of (library variant, environment) pairs with tight timeouts.
# Usage (under gpurun): bash scripts/ab_env.sh "TAG VARIANT [ENV=VAL ...]" ...
# VARIANT base = the product library, else libgroot_b200_VARIANT.so.
mkdir -p gpurun_out
for spec in "$@"; do
  set -- $spec
  tag=$1; v=$2; shift 2
  lib=paper_2511_18297_b200/libgroot_b200.so
  [ "$v" != base ] && lib=paper_2511_18297_b200/libgroot_b200_$v.so
  env GROOT_LIB=$PWD/$lib "$@" timeout 150 python bench.py --no-cpu-baseline --no-side --steps 10 --e2e-steps ${E2E_STEPS:-3} \
    > gpurun_out/abe_$tag.json 2> gpurun_out/abe_$tag.err
  python -c "
import json
try:
    d=json.load(open('gpurun_out/abe_$tag.json')); k=d['kernels']
    print('$tag', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],2), {x:round(v['ms_per_launch'],3) for x,v in k.items() if 'sage' in x or 'l0' in x}, d.get('clocks',{}).get('sm_mhz'))
except Exception as e:
    print('$tag failed', e)"
done
