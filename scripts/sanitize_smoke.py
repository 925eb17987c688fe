"""Small runs of every kernel family for compute-sanitizer (memcheck / racecheck /
synccheck): keyed and materialized forward (tile kernels incl. the tensor-core
head), HD rows, classify_aig, partitions + predict, the LP partitioner,
training, f64 SpMM.

usage: compute-sanitizer --tool memcheck python scripts/sanitize_smoke.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("GROOT_L0_KEYED_MIN_ROWS", "0")  # key the small graphs too
from paper_2511_18297_b200 import api  # noqa: E402

model = api.init_model(7)
for gen, w, b in ((api.gen_csa_multiplier, 16, 3), (api.gen_booth_multiplier, 12, 2), (api.gen_csa_multiplier, 160, 1)):
    c = gen(w)
    g = api.encode(c.aig, c.labels)
    if b > 1:
        g = api.batch(g, b)
    lg = api.forward(model, g)
    p = api.predict_full(model, g)
    print(gen.__name__, w, b, "n", g.n, "acc %.4f" % p.accuracy, "finite", bool(np.isfinite(lg).all()), flush=True)
c = api.gen_csa_multiplier(24)
print("classify_aig", api.classify_aig(model, c.aig, c.labels, 3).accuracy, flush=True)
g = api.batch(api.encode(c.aig, c.labels), 2)
pa = api.partition_multilevel(g, 5)
parts = api.regrow(g, pa)
print("lp + predict", api.edge_cut(g, pa), api.predict(model, g, parts).accuracy, flush=True)
st = api.TrainStats(None, None)
api.train(api.encode(c.aig, c.labels), epochs=3, learning_rate=1e-2, stats=st)
print("train", st.loss, flush=True)
rp = np.array([0, 2, 3, 600], np.uint64)
ci = np.concatenate([[0, 1, 2], np.arange(597) % 3]).astype(np.uint32)
print("spmm f64", float(api.spmm_csr_f64(rp, ci, np.ones(600), np.ones((3, 4)), hd_threshold=512).sum()), flush=True)
# row records with degree > 4 tails (keyed: sparse features; materialized: dense)
from oracle import pyoracle as O  # noqa: E402  (graph construction only)
rng = np.random.default_rng(11)
e = [(int(u), v) for v in range(1, 2000) for u in rng.integers(max(0, v - 60), v, rng.integers(1, 7))]
rp2, ci2 = O.build_csr(2000, np.array(e, np.uint32))
for sparse in (True, False):
    f2 = (rng.random((2000, 4)) < 0.5).astype(np.uint8)
    if sparse:
        f2[:] = 0
        f2[::13, 0] = 1
    g2 = api.EdaGraph.from_host(2000, rp2, ci2, f2, np.zeros(2000, np.uint8))
    print("long rows", "keyed" if sparse else "materialized", bool(np.isfinite(api.forward(model, g2)).all()), flush=True)
print("sanitize smoke done", flush=True)
