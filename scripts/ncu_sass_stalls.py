"""Per-instruction stall attribution from an ncu report's source page (SASS).

usage: python scripts/ncu_sass_stalls.py REPORT [top_k]
Prints the top instructions by warp-stall samples with their dominant stall
reasons, plus shared-memory wavefront / bank-conflict totals.
"""
import csv
import io
import subprocess
import sys


def main(rep, k=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    data = [r for r in rows[2:] if len(r) == len(hdr)]
    col = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]

    def num(r, h):
        try:
            return float(r[col[h]].replace(",", ""))
        except (ValueError, KeyError):
            return 0.0
    tot = sum(num(r, "Warp Stall Sampling (All Samples)") for r in data) or 1.0
    agg = {h: sum(num(r, h) for r in data) for h in stall_cols}
    print("stall totals:", {h[6:]: round(100 * v / tot, 1) for h, v in sorted(agg.items(), key=lambda x: -x[1])[:8]})
    for h in ("L1 Wavefronts Shared", "L1 Wavefronts Shared Ideal", "L1 Wavefronts Shared Excessive"):
        print(h, sum(num(r, h) for r in data))
    data.sort(key=lambda r: -num(r, "Warp Stall Sampling (All Samples)"))
    for r in data[:k]:
        s = num(r, "Warp Stall Sampling (All Samples)")
        top = sorted(((num(r, h), h[6:]) for h in stall_cols), reverse=True)[:2]
        print(f"{100 * s / tot:5.2f}% {r[col['Address']][-5:]} {r[col['Source']].strip()[:60]:60s} "
              + " ".join(f"{n}:{100 * v / max(s, 1):.0f}%" for v, n in top))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
