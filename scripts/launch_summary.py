"""Per-kernel totals of an `ncu --metrics gpu__time_duration.sum --csv` launch list.

usage: python scripts/launch_summary.py LAUNCHES.csv "COMMAND" > profiles/launches_rNN.txt
"""
import collections
import csv
import sys


def main(path, cmd):
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
    hdr = rows[0]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows[1:]:
        if len(r) != len(hdr):
            continue
        name = r[ik].split("(")[0]
        v = float(r[iv].replace(",", "")) * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "nsecond": 1e-6}.get(r[iu], 1e-6)
        tot[name] += v
        cnt[name] += 1
    all_ms = sum(tot.values()) or 1.0
    print(f"# {cmd}")
    print("# per-kernel totals over the captured launches (cold-cache, serialised: compare SHARES, not absolutes)")
    print("# forward step (keyed default) = l0 keys (hd_key, l0_key, dict_finalize, l0_xlat, l0_ids, l0_halo_ids) + l1_xform + 3x(hd_chunk + hd_reduce + sage_tile_kernel) [<3,1> keyed transform-first layer 1, <0,0> layer 2, <1,0> last] + confusion; sage_layer0 launches come from the materialized-layer-0 comparison run")
    for name, ms in tot.most_common():
        print(f"{name[:70]:70s} launches={cnt[name]:4d} total_ms={ms:9.3f} avg_ms={ms / cnt[name]:8.3f} "
              f"share={100 * ms / all_ms:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
