"""racecheck probe: one kernel family on one graph (development aid)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_18297_b200 import api
mode, circ, w, b = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
c = (api.gen_booth_multiplier if circ == "booth" else api.gen_csa_multiplier)(w)
g = api.encode(c.aig, c.labels)
g = api.batch(g, b) if b > 1 else g
if mode == "fwd":
    api.forward(api.init_model(7), g)
else:
    x = np.random.default_rng(0).uniform(-1, 1, (g.n, 32)).astype(np.float32)
    api.spmm_mean(g, x)
print("done", g.n)
