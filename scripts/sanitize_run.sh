#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize_smoke.py
# (keyed path) and memcheck of the materialized path. Usage (under gpurun): bash scripts/sanitize_run.sh TAG
TAG=${1:-r02}
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_smoke.py > gpurun_out/${tool}_$TAG.txt 2>&1
  echo "$tool rc=$?"; tail -2 gpurun_out/${tool}_$TAG.txt
done
GROOT_L0_KEYED=0 timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_smoke.py > gpurun_out/memcheck_materialized_$TAG.txt 2>&1
echo "memcheck materialized rc=$?"; tail -2 gpurun_out/memcheck_materialized_$TAG.txt
