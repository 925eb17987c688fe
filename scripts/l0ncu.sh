#!/bin/bash
# Per-kernel ncu durations of the layer-0 key passes for library variants.
# Usage (under gpurun): bash scripts/l0ncu.sh "TAG VARIANT [ENV=VAL ...]" ...
mkdir -p gpurun_out
for spec in "$@"; do
  set -- $spec
  tag=$1; v=$2; shift 2
  lib=paper_2511_18297_b200/libgroot_b200.so; [ "$v" != base ] && lib=paper_2511_18297_b200/libgroot_b200_$v.so
  env GROOT_LIB=$PWD/$lib "$@" timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"l0_|hd_key|dict_" \
    -c 14 --csv python bench.py --no-cpu-baseline --no-side --steps 1 --warmup 1 --e2e-steps 1 2>/dev/null > gpurun_out/l0ncu_$tag.csv
  python - $tag <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(l for l in open(f'gpurun_out/l0ncu_{sys.argv[1]}.csv') if l.startswith('"'))]
h = rows[0]; ik = h.index('Kernel Name'); iv = h.index('Metric Value')
t = collections.defaultdict(list)
for r in rows[1:]:
    t[r[ik].split('(')[0]].append(float(r[iv].replace(',', '')) / 1e6)
print(sys.argv[1], round(sum(sum(v) / len(v) for v in t.values()), 3), {k: round(sum(v) / len(v), 3) for k, v in t.items()})
PY
done
