"""Generate golden fixtures from the REAL reference build (oracle/_ref).

Run in the build container (needs /root/reference to compile oracle/_ref):

    python tests/golden/make_golden.py

Outputs (committed):
  csa2.npz, csa8.npz  — full arrays: AIG, encode() graph, batch(.,3), topo
                        partitions k=2,3 with regrow/core_subgraphs parts and
                        materialize() CSR, build_plan() of the graph, execute()
                        fp64 output on a seeded dense matrix, predict_full()
                        logits/classes (reference aggregation + restated dense).
  digests.json        — sha256 digests + sizes of the same arrays for larger
                        widths (16, 32, 64 batch 4, 256 batch 1) so the suite
                        checks them without storing megabytes.
  trained_csa8.asg1   — ASG1 model: the reference training recipe (8-bit CSA,
                        100 epochs, lr 1e-3, Adam, seed 7) run through the
                        oracle restatement of train() (src/gnn.cpp:211-255);
                        src/gnn.cpp itself needs Eigen and cannot be compiled.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import pyoracle as O  # noqa: E402
from oracle import pyref as R  # noqa: E402

GRAPH_FIELDS = ["row_ptr", "col_idx", "features", "labels", "degree", "fwd_edges"]


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def graph_arrays(prefix, g):
    return {f"{prefix}{f}": getattr(g, f) for f in GRAPH_FIELDS}


def fixture(width: int, path: str):
    aig, rg = R.gen_csa(width)
    g = rg.to_host()
    out = {"width": np.array(width), "num_inputs": np.array(aig.num_inputs),
           "and_lits": aig.and_lits, "out_lits": aig.out_lits, "aig_labels": aig.labels}
    out.update(graph_arrays("g_", g))
    gb = R.batch(rg, 3).to_host()
    out.update(graph_arrays("b3_", gb))
    for k in (2, 3):
        part = R.topo_chunks(rg, k)
        out[f"topo{k}"] = part
        out[f"topo{k}_crossing"] = np.array(R.crossing_fraction(rg, part, k))
        for mode, wb in (("regrow", True), ("core", False)):
            rp = R.RefParts(rg, part, k, wb)
            out[f"topo{k}_{mode}_footprint"] = np.array(rp.footprint_proxy())
            for p in range(k):
                P = rp.part(p)
                key = f"topo{k}_{mode}_p{p}_"
                out[key + "core"] = P.core_nodes
                out[key + "boundary"] = P.boundary_nodes
                out[key + "edges"] = P.edges
                m = rp.materialize(p).to_host()
                out[key + "m_row_ptr"] = m.row_ptr
                out[key + "m_col_idx"] = m.col_idx
    plan = R.build_plan(g.row_ptr)
    for key in ("hd_rows", "mid_rows", "ld_groups", "units", "perm"):
        out["plan_" + key] = plan[key]
    out["plan_ld_range"] = np.array([plan["ld_row_begin"], plan["ld_row_end"]])
    deg = np.diff(g.row_ptr).astype(np.float64)
    vals = np.repeat(np.where(deg > 0, 1.0 / np.maximum(deg, 1), 0.0), np.diff(g.row_ptr).astype(np.int64))
    rng = np.random.default_rng(0xB00B1E5)
    dense = rng.uniform(-1, 1, size=(g.n, 32))
    out["spmm_dense"] = dense
    out["spmm_out"] = R.plan_execute(plan, g.row_ptr, g.col_idx, vals, dense)
    R.free_plan(plan)
    prm = O.init_model(7)
    out["init7_params"] = prm
    pred, conf, acc, lg = R.predict_full(rg, prm, want_logits=True)
    out["init7_logits"] = lg
    out["init7_pred"] = pred
    out["init7_confusion"] = conf
    out["init7_accuracy"] = np.array(acc)
    np.savez_compressed(path, **out)


def digests():
    res = {}
    for width, b in ((16, 1), (32, 1), (64, 4), (256, 1)):
        aig, rg = R.gen_csa(width)
        if b > 1:
            rg = R.batch(rg, b)
        g = rg.to_host()
        entry = {"n": g.n, "nnz": g.nnz, "edges": g.num_edges,
                 "and_lits": digest(aig.and_lits), "out_lits": digest(aig.out_lits)}
        for f in GRAPH_FIELDS:
            entry[f] = digest(getattr(g, f))
        k = 4
        part = R.topo_chunks(rg, k)
        rp = R.RefParts(rg, part, k, True)
        entry["topo4_regrow"] = [{"core": digest(P.core_nodes), "boundary": digest(P.boundary_nodes),
                                  "edges": digest(P.edges), "n_boundary": int(P.boundary_nodes.shape[0]),
                                  "n_edges": int(P.edges.shape[0])} for P in rp.parts()]
        entry["topo4_footprint"] = rp.footprint_proxy()
        res[f"csa{width}_b{b}"] = entry
    return res


def main():
    R.build()
    fixture(2, os.path.join(HERE, "csa2.npz"))
    fixture(8, os.path.join(HERE, "csa8.npz"))
    with open(os.path.join(HERE, "digests.json"), "w") as f:
        json.dump(digests(), f, indent=1, sort_keys=True)
    g8 = R.gen_csa(8)[1].to_host()
    prm, loss, acc = O.train(g8, epochs=100, lr=1e-3, seed=7)
    O.save_model(os.path.join(HERE, "trained_csa8.asg1"), prm)
    with open(os.path.join(HERE, "trained_csa8.json"), "w") as f:
        json.dump({"recipe": "8-bit CSA, 100 epochs, lr 1e-3, Adam(0.9,0.999,1e-8), seed 7",
                   "final_loss": loss, "final_train_accuracy": acc}, f, indent=1)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
