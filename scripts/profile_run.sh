#!/bin/bash
# One GPU session: smoke, bench, ncu launch list, ncu --set full on the top kernels.
# Usage (under gpurun): bash scripts/profile_run.sh <tag>
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 \
   > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sage_layer_tc_kernel -s 1 -c 1 \
   -o gpurun_out/prof_tc_$TAG -f python scripts/probe_perf.py 1024 16 > gpurun_out/ncu_tc_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"spmm_mean32|hd_mean32|sage_layer0" -c 3 \
   -o gpurun_out/prof_aux_$TAG -f python scripts/probe_perf.py 1024 16 > gpurun_out/ncu_aux_$TAG.log 2>&1
ls -la gpurun_out
