"""Per-role breakdown of one kernel's ncu source page (SASS): instructions
executed per tile and warp-stall samples, by execution-count class.

usage: python scripts/sass_regions.py REPORT KERNEL_INDEX TILES [listing.txt] [kernel regex, default sage_tile]
(KERNEL_INDEX counts launches matching the regex in the report, from 1.)
"""
import csv, io, subprocess, sys
from collections import defaultdict

rep, k, T = sys.argv[1], sys.argv[2], float(sys.argv[3])
kre = sys.argv[5] if len(sys.argv) > 5 else "sage_tile"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--kernel-id", f"::regex:{kre}:{k}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break
    if len(r) == len(hdr):
        data.append(r)
col = {h: i for i, h in enumerate(hdr)}
sc = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]


def num(r, h):
    try:
        return float(r[col[h]].replace(",", ""))
    except (ValueError, KeyError):
        return 0.0


tot = sum(num(r, "Warp Stall Sampling (All Samples)") for r in data) or 1
cls = defaultdict(lambda: [0.0, 0.0, defaultdict(float)])
for r in data:
    e = num(r, "Instructions Executed")
    c = round(e / T) if e else 0
    cls[c][0] += e / T
    cls[c][1] += num(r, "Warp Stall Sampling (All Samples)")
    for h in sc:
        cls[c][2][h[6:]] += num(r, h)
print(f"instructions per tile: {sum(v[0] for v in cls.values()):.0f}")
for c, (ins, smp, st) in sorted(cls.items()):
    if ins < 5 and smp / tot < 0.005:
        continue
    top = sorted(st.items(), key=lambda x: -x[1])[:4]
    print(f"x{c:<4d} instr/tile {ins:7.0f}  samples {100 * smp / tot:5.1f}%  " +
          " ".join(f"{n}:{100 * v / max(smp, 1):.0f}%" for n, v in top))
if len(sys.argv) > 4:
    with open(sys.argv[4], "w") as f:
        for i, r in enumerate(data):
            s = num(r, "Warp Stall Sampling (All Samples)")
            top = sorted(((num(r, h), h[6:]) for h in sc), reverse=True)[:2]
            f.write(f"{i:5d} {100 * s / tot:5.2f} {int(num(r, 'Instructions Executed')):10d} "
                    f"{r[col['Source']].strip()[:70]:70s} " +
                    " ".join(f"{n}:{v / max(s, 1) * 100:.0f}" for v, n in top if v > 0) + "\n")
