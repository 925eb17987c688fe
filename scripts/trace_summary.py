"""Summarise the CTA-0 timeline of the fused layer (GROOT_TRACE=<file>, layer 1).

Row i = tile iteration i of CTA 0; columns = clock64 stamps:
  0 loader: row stage free (TMA issued next)   1 copier: plan + stage ready
  2 copier: halo copies issued                 3 producer (warp 4): loop start
  4 producer: rows + plan landed               5 producer: gather done
  6 producer: A stage free                     7 producer: A stage handed to MMA
  8 MMA: A stage seen                          9 MMA: accumulator free
 10 MMA: issued                               11 epilogue: accumulator ready
 12 epilogue: tile stored
Prints median phase durations and periods in cycles.
"""
import sys

import numpy as np


def warp_totals(t):
    # rows 60..61: per producer warp (4..11) totals over CTA 0's tiles: wait rows, gather, wait A, split+store
    w = t[60:62].reshape(-1)[:32].reshape(8, 4)
    if w.sum() <= 0:
        return
    print("per-warp totals (Mcycles): warp  wait-rows  gather  wait-A  split+store")
    for i in range(8):
        print(f"  {i + 4:2d}  " + "  ".join(f"{x / 1e6:8.3f}" for x in w[i]))


def main(path):
    t = np.loadtxt(path, dtype=np.float64)
    warp_totals(t)
    t = t[:60]
    t = t[(t[:, 3] > 0) & (t[:, 7] > 0)]
    if len(t) < 6:
        print("trace: too few tiles")
        return
    t = t[4:]
    med = lambda x: float(np.median(x))
    rows = [
        ("producer: wait rows", t[:, 4] - t[:, 3]),
        ("producer: gather", t[:, 5] - t[:, 4]),
        ("producer: wait A stage", t[:, 6] - t[:, 5]),
        ("producer: split + TMEM st", t[:, 7] - t[:, 6]),
        ("producer: period", np.diff(t[:, 3])),
        ("rows: TMA issue -> producer sees", t[:, 4] - t[:, 0]),
        ("halo: copier ready -> issued", t[:, 2] - t[:, 1]),
        ("halo: issued -> producer sees", t[:, 4] - t[:, 2]),
        ("mma: handed -> seen", t[:, 8] - t[:, 7]),
        ("mma: wait accumulator", t[:, 9] - t[:, 8]),
        ("mma: issue", t[:, 10] - t[:, 9]),
        ("epilogue: issued -> ready", t[:, 11] - t[:, 10]),
        ("epilogue: drain + store", t[:, 12] - t[:, 11]),
        ("epilogue: period", np.diff(t[:, 11])),
        ("loader: period", np.diff(t[:, 0])),
        ("warp 7: gather", t[:, 14] - t[:, 13]),
        ("warp 7: period", np.diff(t[:, 13])),
        ("warp 7 handed - warp 4 handed", t[:, 15] - t[:, 7]),
        ("warp 7 start - warp 4 start", t[:, 13] - t[:, 3]),
    ]
    for name, x in rows:
        print(f"{name:34s} {med(x):9.0f} cyc")


if __name__ == "__main__":
    main(sys.argv[1])
