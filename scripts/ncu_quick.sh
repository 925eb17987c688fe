#!/bin/bash
# Quick per-kernel DRAM/L2 counters of the standalone SpMM under env knobs.
# usage (under gpurun): bash scripts/ncu_quick.sh "ENV=a" "ENV=b" ...
for cfg in "$@"; do
  env $cfg timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_op_read_hit_rate.pct \
    --clock-control none -k regex:"sage_tile|spmm_mean32" -s 2 -c 1 --csv python scripts/probe_spmm.py 1024 16 2>/dev/null \
    | grep -E "gpu__time|dram__|lts__" | awk -F'","' -v c="$cfg" '{print c, $(NF-2), $NF}'
  env $cfg timeout 300 python scripts/probe_spmm.py 1024 16 | sed "s/^/$cfg /"
done
