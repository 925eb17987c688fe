#!/bin/bash
# ncu --set full of the three 32-wide forward kernels (keyed xform layer 1,
# tensor-core layer, last layer) on the 1024-bit CSA b16 forward, skipping the
# warm-up forward. Usage (under gpurun): bash scripts/ncu_tc.sh TAG [env...]
TAG=${1:-tc}; shift
mkdir -p gpurun_out
env "$@" timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sage_tile_kernel" -s 3 -c 3 \
   -o gpurun_out/prof_$TAG -f python scripts/probe_perf.py 1024 16 > gpurun_out/ncu_$TAG.log 2>&1
tail -3 gpurun_out/ncu_$TAG.log
