"""Small end-to-end pass over every device kernel family (keyed layer 0 by default;
GROOT_L0_KEYED=0 for the materialized one), for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool memcheck python scripts/sanitize_smoke.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_18297_b200 import api  # noqa: E402

os.environ.setdefault("GROOT_L0_KEYED_MIN_ROWS", "0")  # key these small graphs too

prm_model = api.init_model(7)
for maker, w, b in ((api.gen_csa_multiplier, 16, 3), (api.gen_booth_multiplier, 12, 2), (api.gen_csa_multiplier, 160, 1)):
    c = maker(w)
    g = api.batch(api.encode(c.aig, c.labels), b) if b > 1 else api.encode(c.aig, c.labels)
    lg = api.forward(prm_model, g)
    pred = api.predict_full(prm_model, g)
    x = np.random.default_rng(0).uniform(-1, 1, (g.n, 32)).astype(np.float32)
    api.spmm_mean(g, x)
    pa = api.partition_topo_chunks(g, 3)
    parts = api.regrow(g, pa)
    api.predict(prm_model, g, parts)
    sub = api.materialize(g, parts, 1)
    api.forward(prm_model, sub)
    api.classify_aig(prm_model, c.aig, c.labels, 3)  # tile-aligned batch, periodic plan, split last layer
    print(maker.__name__, w, b, "n", g.n, "acc", round(pred.accuracy, 4), "finite", bool(np.isfinite(lg).all()))
print("sanitize smoke done")
