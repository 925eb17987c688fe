import sys; sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2511_18297_b200 import api
from oracle import pyoracle as O
c = api.gen_booth_multiplier(64)
g = api.batch(api.encode(c.aig, c.labels), 4)
rp = g.row_ptr; deg = np.diff(rp)
print("n", g.n, "max deg", deg.max(), "deg>=128:", (deg >= 128).sum(), "hist top", np.bincount(deg)[-5:])
prm = O.init_model(7)
lg = api.forward(api.Model.from_params(prm), g)
print("ok", lg.shape)
