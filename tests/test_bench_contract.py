"""bench.py output contract: one JSON line with the keys the driver reads.

CPU: the reference arm (`--impl reference`, the compiled reference path in
oracle/_ref) at the 8-bit config. GPU: our arm at a small config, checking
every contract key (value, e2e with host<->device bytes, roofline, clocks,
gpu_launches) and that the numbers are self-consistent.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config")


def run_bench(*args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    from oracle import pyref
    if not pyref.available():
        pytest.skip("reference build (oracle/_ref) not available")
    d = run_bench("--impl", "reference", "--width", "8", "--batch", "1", "--steps", "2", "--warmup", "1")
    assert d["impl"] == "reference"
    for k in BASE_KEYS:
        assert k in d, k
    assert d["value"] > 0 and d["unit"] == "edges/s" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_our_arm_line():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    d = run_bench("--width", "64", "--batch", "4", "--steps", "3", "--warmup", "3", "--no-cpu-baseline")
    for k in BASE_KEYS + ("e2e", "roofline", "clocks", "gpu_launches", "spmm", "kernels"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] >= 3 and d["scaling"] == "weak"
    assert d["roofline"]["kernel"] in d["kernel_rooflines"] and d["like_for_like"] is None
    assert "workload" in d["config"]
    edges = d["config"]["edges_per_gpu"]
    assert abs(d["value"] - edges / (d["ms_per_step"] * 1e-3)) <= 1e-6 * d["value"]
    e2e = d["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] >= d["config"]["nodes_per_gpu"]
    roof = d["roofline"]
    assert roof["bound"] == "hbm" and roof["unit"] == "GB/s" and roof["peak"] > 0
    assert abs(roof["frac"] - roof["achieved"] / roof["peak"]) < 1e-9
    assert d["gpu_launches"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
