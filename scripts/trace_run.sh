#!/bin/bash
# CTA-0 timelines of the tile kernels (trace build: scripts/variant.sh trace -DGROOT_TRACE_BUILD).
# Usage (under gpurun): bash scripts/trace_run.sh TAG [layers...]
TAG=${1:-t}; shift
for L in "${@:-1 2 3}"; do
  GROOT_LIB=$PWD/paper_2511_18297_b200/libgroot_b200_trace.so GROOT_TRACE=gpurun_out/trace_${TAG}_L$L.txt GROOT_TRACE_LAYER=$L \
    timeout 300 python scripts/probe_perf.py 1024 16 > /dev/null 2>&1
  echo "== layer $L"; python scripts/trace_summary.py gpurun_out/trace_${TAG}_L$L.txt
done
