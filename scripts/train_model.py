"""Train a GraphSAGE classifier on the device (csrc/train.cu) and evaluate it:
per-width accuracy of predict_full on CSA multipliers, and whether the verifier
(backward_rewrite) proves the multipliers from the predicted classes.

usage: python scripts/train_model.py OUT.asg1 --width 16 --epochs 2000 --lr 1e-2
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_18297_b200 import api  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("out")
    p.add_argument("--width", type=int, default=16)
    p.add_argument("--copies", type=int, default=1)
    p.add_argument("--epochs", type=int, default=2000)
    p.add_argument("--lr", type=float, default=1e-2)
    p.add_argument("--seed", type=int, default=7)
    p.add_argument("--booth", type=int, default=0, help="also train on a Booth AIG of this width (0: no)")
    p.add_argument("--verify", type=str, default="8,16,32")
    a = p.parse_args()
    c = api.gen_csa_multiplier(a.width)
    g = api.encode(c.aig, c.labels)
    if a.copies > 1:
        g = api.batch(g, a.copies)
    t0 = time.time()
    st = api.TrainStats(None, None)
    model = api.train(g, epochs=a.epochs, learning_rate=a.lr, seed=a.seed, stats=st)
    dt = time.time() - t0
    api.save_model(a.out, model)
    res = {"recipe": f"{a.width}-bit CSA x{a.copies}, {a.epochs} epochs, lr {a.lr}, Adam(0.9,0.999,1e-8), seed {a.seed}, "
                     f"device fp64 (csrc/train.cu)", "train_s": dt, "final_loss": float(st.loss[-1]),
           "final_train_accuracy": float(st.accuracy[-1]), "accuracy": {}, "verify": {}}
    for w in (8, 16, 32, 64, 256, 1024):
        cw = api.gen_csa_multiplier(w)
        pr = api.predict_full(model, api.encode(cw.aig, cw.labels))
        res["accuracy"][f"csa{w}"] = pr.accuracy
        if str(w) in a.verify.split(","):
            t1 = time.time()
            rep = api.backward_rewrite(cw.aig, pr.labels, w)
            res["verify"][f"csa{w}"] = {"equivalent": rep.equivalent, "inconclusive": rep.inconclusive,
                                        "shortcuts": rep.shortcut_count, "fallbacks": rep.fallback_count,
                                        "seconds": time.time() - t1}
    for w in (16, 64):
        cb = api.gen_booth_multiplier(w)
        res["accuracy"][f"booth{w}"] = api.predict_full(model, api.encode(cb.aig, cb.labels)).accuracy
    print(json.dumps(res))
    with open(os.path.splitext(a.out)[0] + ".json", "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
