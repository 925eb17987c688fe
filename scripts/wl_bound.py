"""Accuracy ceiling of any depth-L message-passing GNN on the reference's node
features: Weisfeiler-Lehman colour refinement (own colour + multiset of the
neighbours' colours, injective) from the 4 encode features; nodes of one colour
after L rounds are indistinguishable to every L-layer GNN whose aggregation is
a function of the neighbour multiset (GraphSAGE-mean is weaker still), so the
best per-node accuracy is the sum over colours of the majority label count.

usage: python scripts/wl_bound.py WIDTH [DEPTH]   (CSA multiplier, oracle encode)
"""
import os
import sys
from collections import Counter, defaultdict

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import pyoracle as O  # noqa: E402


def wl_bound(g, depth):
    rp = g.row_ptr.astype(np.int64)
    ci = g.col_idx.astype(np.int64)
    n = g.n
    lab = np.asarray(g.labels)
    feat = np.asarray(g.features).reshape(n, 4)
    col = [hash(tuple(feat[v])) for v in range(n)]
    out = []
    for _ in range(depth):
        col = [hash((col[v], tuple(sorted(col[u] for u in ci[rp[v]:rp[v + 1]])))) for v in range(n)]
        by = defaultdict(Counter)
        for v in range(n):
            by[col[v]][lab[v]] += 1
        out.append((len(by), sum(c.most_common(1)[0][1] for c in by.values()) / n))
    return out


if __name__ == "__main__":
    w = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    d = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    for depth, (colours, acc) in enumerate(wl_bound(O.encode(O.gen_csa(w)), d), 1):
        print(f"CSA {w}: depth {depth}: {colours} colours, best accuracy {acc:.4f}")
