"""Build profiles/ncu_summary.json from `ncu --set full` reports.

usage: python scripts/make_profile_summary.py ROUND OUT.json REPORT [REPORT ...]

Per kernel (first capture of each name): duration, DRAM bytes read/written
(the `traffic` figure bench.py reports), throughput percentages, launch
shape, and for the fused layer the top SASS lines by warp-stall samples.
"""
import json
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_summary as N  # noqa: E402

CONFIG = "csa1024_b16"  # the workload the reports were captured on (bench.py cfg_key)
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def short_name(k):
    m = re.search(r"sage_tile_kernel<(\d)(?:, (true|false|0|1))?>", k) or re.search(r"sage_tile_kernelILi(\d)E(?:Lb(\d)E)?", k)
    if m:  # template modes: 0 layer, 1 last layer, 2 standalone SpMM; keyed (entry-table input) variants
        mode, keyed = m.group(1), m.group(2) in ("true", "1")
        base = {"0": "sage_layer_tc", "1": "sage_layer_tc_last", "2": "spmm_mean32", "3": "sage_layer1_xform"}[mode]
        return base + ("_keyed" if keyed and mode == "0" else "")
    if "tile_plan_kernel" in k:
        return "tile_plan"
    for key in ("sage_layer0", "hd_mean_feat", "hd_mean32", "confusion", "spmm_mean32", "spmm_generic", "naive_layer"):
        if key in k:
            return key
    return k.split("(")[0].split()[-1]


def val(m, key, scale=False):
    e = m.get(key)
    if not isinstance(e, dict):
        return None
    try:
        v = float(str(e["value"]).replace(",", ""))
    except ValueError:
        return None
    return v * UNIT.get(e.get("unit", ""), 1.0) if scale else v


def main(rnd, out, reports):
    kernels = {}
    for rep in reports:
        stalls = {short_name(s["kernel"]): s["top"] for s in N.top_sass(rep, 8)}
        for m in N.raw(rep):
            kname = m["kernel"]
            name = short_name(kname)
            if name in kernels:
                continue
            rd, wr = val(m, "dram__bytes_read.sum", True), val(m, "dram__bytes_write.sum", True)
            e = {
                "duration_ms": val(m, "gpu__time_duration.sum"),
                "dram_read_bytes": rd,
                "dram_write_bytes": wr,
                "dram_bytes_per_launch": (rd or 0) + (wr or 0),
                "dram_throughput_pct": val(m, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                "lts_throughput_pct": val(m, "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
                "l1tex_throughput_pct": val(m, "l1tex__throughput.avg.pct_of_peak_sustained_elapsed"),
                "tensor_pipe_active_pct": val(m, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
                "warps_active_pct": val(m, "sm__warps_active.avg.pct_of_peak_sustained_active"),
                "registers": val(m, "launch__registers_per_thread"),
                "grid": val(m, "launch__grid_size"),
                "block": val(m, "launch__block_size"),
                "source": os.path.basename(rep),
            }
            if name.startswith("sage_layer_tc") and name in stalls:
                e["top_stalls"] = stalls[name]
            kernels[name] = e
    res = {"round": rnd, "source": "ncu --set full --clock-control none (" + ", ".join(os.path.basename(r) for r in reports)
           + "); 1024-bit CSA b16 graph", "kernels": kernels}
    # bench.py reads <kernel>.dram_bytes_per_launch at the top level
    for k in ("sage_layer_tc", "sage_layer_tc_last"):
        if k in kernels:
            res[k] = {"dram_bytes_per_launch": kernels[k]["dram_bytes_per_launch"]}
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    # measured DRAM bytes per launch for bench.py's `traffic` (profiles/ncu_traffic.json),
    # keyed "<config>:<profiler scope>"; multi-kernel scopes are the sum of their kernels'
    # mean bytes per launch
    per = {}
    for rep in reports:
        for m in N.raw(rep):
            name = short_name(m["kernel"])
            rd, wr = val(m, "dram__bytes_read.sum", True), val(m, "dram__bytes_write.sum", True)
            per.setdefault(name, []).append((rd or 0) + (wr or 0))
    mean = {k: sum(v) / len(v) for k, v in per.items()}
    scopes = {
        "l0_keys": ["hd_key_kernel", "l0_key_kernel", "l0_key_tile_kernel", "dict_finalize_kernel", "l0_xlat_kernel", "l0_ids_kernel",
                    "l0_halo_ids_kernel", "l0_hd_ids_kernel"],
        "hd_mean32": ["hd_chunk_kernel", "hd_reduce_kernel"],
        "spmm_mean32": ["spmm_mean32", "hd_chunk_kernel", "hd_reduce_kernel"],
    }
    traffic = {}
    for k, v in mean.items():
        if k in ("sage_layer_tc", "sage_layer_tc_last", "sage_layer1_xform", "sage_layer_tc_keyed", "sage_layer0",
                 "confusion", "tile_plan"):
            traffic[f"{CONFIG}:{k}"] = v
    for scope, members in scopes.items():
        if any(m in mean for m in members):
            traffic[f"{CONFIG}:{scope}"] = sum(mean.get(m, 0.0) for m in members)
    tpath = os.path.join(os.path.dirname(out), "ncu_traffic.json")
    with open(tpath, "w") as f:
        json.dump(dict(sorted(traffic.items()), _source=res["source"]), f, indent=1)


if __name__ == "__main__":
    main(int(sys.argv[1]), sys.argv[2], sys.argv[3:])
