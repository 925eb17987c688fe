#!/bin/bash
# A/B of library variants (scripts/variant.sh) on the bench's device forward:
# bash scripts/ab_variants.sh base nohead hint ...   ("base" = the product library)
for v in "$@"; do
  lib=paper_2511_18297_b200/libgroot_b200.so
  [ "$v" != base ] && lib=paper_2511_18297_b200/libgroot_b200_$v.so
  for rep in 1 2; do
    GROOT_LIB=$PWD/$lib timeout 600 python bench.py --no-cpu-baseline --no-side --steps 10 --e2e-steps 3 > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
    python -c "
import json,sys; d=json.load(open('gpurun_out/ab_$v.json')); k=d['kernels']
print('$v', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],2), {x:round(v['ms_per_launch'],3) for x,v in k.items() if 'sage' in x or 'l0' in x})" || tail -3 gpurun_out/ab_$v.err
  done
done
