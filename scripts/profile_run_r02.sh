#!/bin/bash
# One GPU session: tests, smoke, bench (+reference arm), ncu launch list of the
# bench command, ncu --set full of every forward kernel (keyed default path and
# the materialized path) and of the standalone SpMM.
# Usage (under gpurun): bash scripts/profile_run_r02.sh <tag> [all]; the
# materialized-path and SpMM captures: bash scripts/profile_run_r02.sh <tag> ncu2
TAG=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_$TAG.txt 2>&1
nproc >> gpurun_out/gpu_$TAG.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/gpu_$TAG.txt
if [ "$2" = ncu2 ]; then
GROOT_L0_KEYED=0 timeout 900 ncu --set full --clock-control none --import-source on -k "regex:sage_layer0|sage_tile" -s 0 -c 4 \
   -o gpurun_out/prof_mat_$TAG -f python scripts/probe_perf.py 1024 16 > gpurun_out/ncu_mat_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sage_tile|hd_chunk" -s 3 -c 2 \
   -o gpurun_out/prof_spmm_$TAG -f python scripts/probe_spmm.py 1024 16 > gpurun_out/ncu_spmm_$TAG.log 2>&1
exit 0
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rf -s --durations=25 > gpurun_out/tests_$TAG.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
   --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
   > gpurun_out/launches_bench_$TAG.json 2>&1
KSEL='regex:sage_tile|sage_layer0|hd_chunk|hd_reduce|confusion|tile_plan|l0_key|l0_halo|l0_ids|hd_key'
timeout 900 ncu --set full --clock-control none --import-source on -k "$KSEL" -s 0 -c 18 \
   -o gpurun_out/prof_$TAG -f python scripts/probe_perf.py 1024 16 > gpurun_out/ncu_$TAG.log 2>&1
[ "$2" = all ] || { ls -la gpurun_out | tail -20; exit 0; }  # the rest in a second call (gpurun_out <= 64 MiB)
GROOT_L0_KEYED=0 timeout 900 ncu --set full --clock-control none --import-source on -k "regex:sage_layer0|sage_tile" -s 0 -c 4 \
   -o gpurun_out/prof_mat_$TAG -f python scripts/probe_perf.py 1024 16 > gpurun_out/ncu_mat_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sage_tile|hd_chunk" -s 3 -c 2 \
   -o gpurun_out/prof_spmm_$TAG -f python scripts/probe_spmm.py 1024 16 > gpurun_out/ncu_spmm_$TAG.log 2>&1
ls -la gpurun_out | tail -30
