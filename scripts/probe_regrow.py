"""Time topo k + regrow + predict on the 1024-bit CSA b16 graph (host wall clock per stage)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_18297_b200 import api
k = int(sys.argv[1]) if len(sys.argv) > 1 else 64
c = api.gen_csa_multiplier(1024)
g = api.batch(api.encode(c.aig, c.labels), 16)
model = api.init_model(7)
for rep in range(3):
    t0 = time.perf_counter(); pa = api.partition_topo_chunks(g, k)
    t1 = time.perf_counter(); parts = api.regrow(g, pa)
    t2 = time.perf_counter(); pred = api.predict(model, g, parts)
    t3 = time.perf_counter()
    print(f"k={k} topo {1e3*(t1-t0):.1f} ms regrow {1e3*(t2-t1):.1f} ms predict {1e3*(t3-t2):.1f} ms", flush=True)
    del parts, pa, pred
