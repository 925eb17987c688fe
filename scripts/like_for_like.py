"""Like-for-like pair at BASELINE config 5 partitioned: the whole
1024-bit CSA b16 graph, topo k partitions, regrow, predict over every part --
the reference's own compiled code on all host threads vs the device path,
same inputs, same k, same model. Prints one JSON object.

usage: python scripts/like_for_like.py [--width 1024] [--batch 16] [--k 128]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import pyoracle as O  # noqa: E402
from oracle import pyref as R  # noqa: E402
from paper_2511_18297_b200 import api  # noqa: E402

MODEL = os.path.join(ROOT, "tests", "golden", "trained_csa8.asg1")


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--width", type=int, default=1024)
    p.add_argument("--batch", type=int, default=16)
    p.add_argument("--k", type=int, default=128)
    a = p.parse_args()
    prm = O.load_model(MODEL)[0]
    res = {"workload": f"{a.width}-bit CSA b{a.batch}, topo k={a.k}, regrow, predict over all parts",
           "cores": R.default_workers()}
    # --- reference (compiled sources, oracle/_ref): gen, encode, batch, topo, regrow, predict
    t0 = time.perf_counter()
    _, rg = R.gen_csa(a.width)
    rb = R.batch(rg, a.batch) if a.batch > 1 else rg
    t1 = time.perf_counter()
    part = R.topo_chunks(rb, a.k)
    rparts = R.RefParts(rb, part, a.k, True)
    t2 = time.perf_counter()
    n = rb.sizes()[0]
    rpred = np.zeros(n, np.uint8)
    R.predict_parts(rparts, 0, a.k, prm, pred=rpred)
    t3 = time.perf_counter()
    E = rb.sizes()[2]
    res["reference"] = {"graph_build_s": t1 - t0, "topo_regrow_s": t2 - t1, "predict_s": t3 - t2,
                        "chain_s": t3 - t1, "edges_per_s_chain": E / (t3 - t1), "edges_per_s_predict": E / (t3 - t2)}
    del rparts
    # --- device: same chain through the C ABI (host arrays in, host classes out)
    model = api.Model.from_params(prm)
    c = api.gen_csa_multiplier(a.width)
    g = api.batch(api.encode(c.aig, c.labels), a.batch)
    api.predict(model, g, api.regrow(g, api.partition_topo_chunks(g, a.k)))  # warm-up
    t0 = time.perf_counter()
    pa = api.partition_topo_chunks(g, a.k)
    parts = api.regrow(g, pa)
    t1 = time.perf_counter()
    pred = api.predict(model, g, parts)
    t2 = time.perf_counter()
    res["device"] = {"topo_regrow_s": t1 - t0, "predict_s": t2 - t1, "chain_s": t2 - t0,
                     "edges_per_s_chain": E / (t2 - t0), "edges_per_s_predict": E / (t2 - t1)}
    res["edges"] = int(E)
    res["ratio_chain"] = res["device"]["edges_per_s_chain"] / res["reference"]["edges_per_s_chain"]
    res["ratio_predict"] = res["device"]["edges_per_s_predict"] / res["reference"]["edges_per_s_predict"]
    res["classes_equal"] = bool(np.array_equal(pred.labels, rpred))
    res["class_mismatches"] = int((pred.labels != rpred).sum())
    print(json.dumps(res))


if __name__ == "__main__":
    main()
