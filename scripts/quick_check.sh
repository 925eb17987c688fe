#!/bin/bash
# Development loop on the GPU box: key parity tests, then two short bench runs
# (device-resident and e2e ms, per-kernel ms). Usage: bash scripts/quick_check.sh [extra pytest args]
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_keyed_layer0.py tests/test_gpu_parity.py -x -q -k "keyed or forward or classify" "$@" 2>&1 | tail -2
for i in 1 2; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bk.json 2> gpurun_out/bk.err
  python - <<'PY'
import json
try:
    d = json.loads(open("gpurun_out/bk.json").readline())
    print(round(d["value"] / 1e9, 3), "G edges/s", round(d["ms_per_step"], 3), "ms; e2e", round(d["e2e"]["ms_per_step"], 3), "ms")
    print({k: round(v["ms_per_step"], 3) for k, v in d["kernels"].items()})
except Exception as e:
    print("bench failed:", e, open("gpurun_out/bk.err").read()[-600:])
PY
done
