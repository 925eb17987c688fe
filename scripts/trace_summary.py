"""Summarise the CTA-0 timeline of the fused layer (GROOT_TRACE=<file>, layer 1).

Row i = tile i of CTA 0; columns (clock64 of the recording thread):
  0..5   first producer warp, lane 0, consume(tile): start, -, -, mean done,
         A stage free (empty), stage handed over (full arrive)
  6..9   same thread, issue(tile): start, input tile landed, col_idx ready,
         neighbour loads issued
  10..13 MMA thread: start, full seen, accumulator free, MMAs issued
  14..15 epilogue warp 0: accumulator ready, tile stored
Prints median phase durations in cycles and the tile period.
"""
import sys

import numpy as np


def main(path):
    t = np.loadtxt(path, dtype=np.float64)
    t = t[(t[:, 0] > 0) & (t[:, 5] > 0)]
    if len(t) < 4:
        print("trace: too few tiles")
        return
    t = t[2:]  # skip warm-up tiles
    med = lambda x: float(np.median(x))
    rows = [
        ("issue: wait input tile", t[:, 7] - t[:, 6]),
        ("issue: row_ptr/col_idx", t[:, 8] - t[:, 7]),
        ("issue: neighbour loads", t[:, 9] - t[:, 8]),
        ("consume: sum+mean", t[:, 3] - t[:, 0]),
        ("consume: wait A stage", t[:, 4] - t[:, 3]),
        ("consume: TMEM store+arrive", t[:, 5] - t[:, 4]),
        ("producer: consume period", np.diff(t[:, 0])),
        ("mma: wait full", t[:, 11] - t[:, 10]),
        ("mma: wait acc", t[:, 12] - t[:, 11]),
        ("mma: issue", t[:, 13] - t[:, 12]),
        ("mma: full -> epi ready", t[:, 14] - t[:, 11]),
        ("epilogue: drain+store", t[:, 15] - t[:, 14]),
        ("epilogue: period", np.diff(t[:, 14])),
    ]
    for name, x in rows:
        print(f"{name:28s} {med(x):9.0f} cyc")


if __name__ == "__main__":
    main(sys.argv[1])
