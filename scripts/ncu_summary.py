"""Summarise ncu reports: per-kernel key metrics + top stall sites.

    python scripts/ncu_summary.py gpurun_out/prof_tc_r01.ncu-rep [...] > profiles/x.json
"""
import csv
import io
import json
import re
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_wait", "smsp__pcsamp_warps_issue_stalled_barrier",
    "smsp__pcsamp_warps_issue_stalled_lg_throttle", "smsp__pcsamp_warps_issue_stalled_mio_throttle",
    "smsp__pcsamp_warps_issue_stalled_short_scoreboard", "smsp__pcsamp_warps_issue_stalled_selected",
    "smsp__pcsamp_warps_issue_stalled_not_selected", "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle",
    "smsp__pcsamp_warps_issue_stalled_sleeping", "smsp__pcsamp_warps_issue_stalled_branch_resolving",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    v = r[i]
                d[k] = {"value": v, "unit": units[i]}
        res.append(d)
    return res


def top_sass(rep, k=12):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    blocks, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = {"kernel": r[1], "rows": []}
            blocks.append(cur)
        elif r and r[0] == "Address":
            cur["hdr"] = r
        elif cur is not None and "hdr" in cur and len(r) == len(cur["hdr"]):
            cur["rows"].append(r)
    res = []
    for b in blocks:
        h = b["hdr"]
        isamp, isrc = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
        data = []
        for r in b["rows"]:
            try:
                data.append((int(r[isamp]), r[isrc].strip()))
            except ValueError:
                pass
        tot = sum(d[0] for d in data) or 1
        res.append({"kernel": b["kernel"], "samples": tot,
                    "top": [{"pct": round(100 * s / tot, 2), "sass": src} for s, src in sorted(data, reverse=True)[:k]]})
    return res


def main():
    out = {}
    for rep in sys.argv[1:]:
        out[rep] = {"metrics": raw(rep), "stalls": top_sass(rep)}
    json.dump(out, sys.stdout, indent=1)


if __name__ == "__main__":
    main()
