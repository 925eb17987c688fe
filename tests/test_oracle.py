"""Pin the oracle restatement (oracle/oracle.cpp) before trusting it.

(1) Against golden fixtures produced by the REAL reference build (always runs).
(2) Against the reference library itself, when oracle/_ref is loadable.
(3) SPEC known answers: 2-bit appendix, degree_sort, HD chunking, regrow laws.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import pyoracle as O

FIELDS = ["row_ptr", "col_idx", "features", "labels", "degree", "fwd_edges"]


def _digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module", params=[2, 8])
def fx(request, golden_dir):
    return np.load(os.path.join(golden_dir, f"csa{request.param}.npz"))


def test_gen_csa_matches_golden(fx):
    a = O.gen_csa(int(fx["width"]))
    assert a.num_inputs == int(fx["num_inputs"])
    np.testing.assert_array_equal(a.and_lits, fx["and_lits"])
    np.testing.assert_array_equal(a.out_lits, fx["out_lits"])
    np.testing.assert_array_equal(a.labels, fx["aig_labels"])


def test_encode_and_batch_match_golden(fx):
    g = O.encode(O.gen_csa(int(fx["width"])))
    for f in FIELDS:
        np.testing.assert_array_equal(getattr(g, f), fx["g_" + f], err_msg=f)
    b = O.batch(g, 3)
    for f in FIELDS:
        np.testing.assert_array_equal(getattr(b, f), fx["b3_" + f], err_msg=f)


def test_partition_regrow_materialize_match_golden(fx):
    g = O.encode(O.gen_csa(int(fx["width"])))
    for k in (2, 3):
        part = O.topo_chunks(g.n, k)
        np.testing.assert_array_equal(part, fx[f"topo{k}"])
        assert O.crossing_fraction(g, part) == float(fx[f"topo{k}_crossing"])
        for mode, wb in (("regrow", True), ("core", False)):
            parts = O.regrow(g, part, k, wb)
            assert O.footprint_proxy(parts) == int(fx[f"topo{k}_{mode}_footprint"])
            for p, P in enumerate(parts):
                key = f"topo{k}_{mode}_p{p}_"
                np.testing.assert_array_equal(P.core_nodes, fx[key + "core"])
                np.testing.assert_array_equal(P.boundary_nodes, fx[key + "boundary"])
                np.testing.assert_array_equal(P.edges, fx[key + "edges"])
                m = O.materialize(g, P)
                np.testing.assert_array_equal(m.row_ptr, fx[key + "m_row_ptr"])
                np.testing.assert_array_equal(m.col_idx, fx[key + "m_col_idx"])


def test_plan_and_spmm_match_golden(fx):
    g = O.encode(O.gen_csa(int(fx["width"])))
    plan = O.build_plan(g.row_ptr)
    for key in ("hd_rows", "mid_rows", "ld_groups", "units", "perm"):
        np.testing.assert_array_equal(plan[key], fx["plan_" + key], err_msg=key)
    deg = np.diff(g.row_ptr)
    vals = np.repeat(np.where(deg > 0, 1.0 / np.maximum(deg, 1), 0.0), deg.astype(np.int64))
    out = O.plan_execute(plan, g.row_ptr, g.col_idx, vals, fx["spmm_dense"])
    np.testing.assert_array_equal(out, fx["spmm_out"])  # bitwise: same accumulation order
    O.free_plan(plan)


def test_forward_matches_golden(fx):
    g = O.encode(O.gen_csa(int(fx["width"])))
    prm = O.init_model(7)
    np.testing.assert_array_equal(prm, fx["init7_params"])
    pred, conf, acc, lg = O.predict_full(g, prm)
    np.testing.assert_array_equal(lg, fx["init7_logits"])
    np.testing.assert_array_equal(pred, fx["init7_pred"])
    np.testing.assert_array_equal(conf, fx["init7_confusion"])
    assert acc == float(fx["init7_accuracy"])


def test_digests_larger_widths(golden_dir):
    with open(os.path.join(golden_dir, "digests.json")) as f:
        dig = json.load(f)
    for name, entry in dig.items():
        w, b = name[3:].split("_b")
        g = O.encode(O.gen_csa(int(w)))
        g = O.batch(g, int(b))
        assert (g.n, g.nnz, g.num_edges) == (entry["n"], entry["nnz"], entry["edges"])
        for f in FIELDS:
            assert _digest(getattr(g, f)) == entry[f], (name, f)
        part = O.topo_chunks(g.n, 4)
        parts = O.regrow(g, part, 4, True)
        for P, e in zip(parts, entry["topo4_regrow"]):
            assert _digest(P.core_nodes) == e["core"]
            assert _digest(P.boundary_nodes) == e["boundary"]
            assert _digest(P.edges) == e["edges"]
        assert O.footprint_proxy(parts) == entry["topo4_footprint"]


def test_spec_known_answers():
    g = O.encode(O.gen_csa(2))
    assert g.n == 19
    f = g.features
    assert f[5].tolist() == [1, 1, 0, 0] and f[10].tolist() == [1, 1, 1, 1]
    assert f[1].tolist() == [0, 0, 0, 0] and f[15].tolist() == [0, 0, 1, 1]
    lab = g.labels
    assert lab[[10, 14]].tolist() == [2, 2] and lab[[8, 12]].tolist() == [1, 1]
    assert lab[[1, 2, 3, 4]].tolist() == [4] * 4 and lab[[15, 16, 17, 18]].tolist() == [0] * 4
    # degree_sort [3,1,2] -> perm [1,2,0]
    perm, _ = O.degree_sort(np.array([0, 3, 4, 6], np.uint64))
    assert perm.tolist() == [1, 2, 0]
    # one row of degree 2048 -> 32 chunks of 64; degree 1000 -> 24x31 then 8x32
    for d, expect in ((2048, [64] * 32), (1000, [31] * 24 + [32] * 8)):
        plan = O.build_plan(np.array([0, d], np.uint64))
        u = plan["units"]
        assert (u[:, 4] - u[:, 3]).tolist() == expect
        O.free_plan(plan)
    # topo k=2 on 2-bit: {0..8},{9..18} (SPEC drift noted in SURVEY 0.1.6)
    assert O.topo_chunks(19, 2).tolist() == [0] * 9 + [1] * 10
    parts = O.regrow(g, O.topo_chunks(19, 2), 2)
    assert parts[0].boundary_nodes.tolist() == [9, 10, 11, 12, 13, 15]
    assert parts[1].boundary_nodes.tolist() == [2, 4, 5, 6, 7, 8]
    assert O.crossing_fraction(g, O.topo_chunks(19, 2)) == 1 / 3
    assert O.footprint_proxy(parts) == 2560


def test_regrow_laws_random_graphs():
    """SPEC acceptance #4: brute-force B_p on 50 random graphs, n <= 200."""
    rng = np.random.default_rng(11)
    for t in range(50):
        n = int(rng.integers(2, 200))
        E = int(rng.integers(0, 3 * n))
        edges = rng.integers(0, n, size=(E, 2)).astype(np.uint32)
        rp, ci = O.build_csr(n, edges)
        g = O.HostGraph(n, rp, ci, np.zeros((n, 4), np.uint8), np.zeros(n, np.uint8),
                        np.diff(rp).astype(np.uint32), edges)
        k = int(rng.integers(1, min(n, 8) + 1))
        part = rng.integers(0, k, size=n).astype(np.uint32)
        parts = O.regrow(g, part, k)
        count = np.zeros(E, np.int64)
        for p, P in enumerate(parts):
            core = set(np.nonzero(part == p)[0].tolist())
            assert P.core_nodes.tolist() == sorted(core)
            brute = sorted({int(u) for v in core for u in ci[rp[v]:rp[v + 1]] if int(u) not in core})
            assert P.boundary_nodes.tolist() == brute
        for (u, v) in edges.tolist():
            count_uv = 1 if part[u] == part[v] else 2
            assert count_uv in (1, 2)
        total = sum(P.edges.shape[0] for P in parts)
        cross = int((part[edges[:, 0]] != part[edges[:, 1]]).sum()) if E else 0
        assert total == E + cross


# ---------------------------------------------------------------------------
# (2) the restatement against the reference library itself (oracle/_ref)
# ---------------------------------------------------------------------------
def _ref():
    from oracle import pyref as R
    if not R.available():
        pytest.skip("oracle/_ref (the compiled reference) is not built")
    return R


@pytest.mark.parametrize("width,copies", [(3, 2), (16, 1), (33, 3), (64, 4), (128, 2)])
def test_restatement_vs_reference_graph_stages(width, copies):
    """gen_csa/encode/batch/topo/regrow/core_subgraphs/materialize/crossing, bit-exact."""
    R = _ref()
    raig, rg = R.gen_csa(width)
    a = O.gen_csa(width)
    np.testing.assert_array_equal(a.and_lits, raig.and_lits)
    np.testing.assert_array_equal(a.out_lits, raig.out_lits)
    np.testing.assert_array_equal(a.labels, raig.labels)
    g = O.batch(O.encode(a), copies) if copies > 1 else O.encode(a)
    rb = R.batch(rg, copies) if copies > 1 else rg
    for f in FIELDS:
        np.testing.assert_array_equal(getattr(g, f), rb.field(f), err_msg=f)
    for k in (1, 2, 5, 16):
        part = O.topo_chunks(g.n, k)
        np.testing.assert_array_equal(part, R.topo_chunks(rb, k))
        assert O.crossing_fraction(g, part) == R.crossing_fraction(rb, part, k)
        for wb in (True, False):
            parts = O.regrow(g, part, k, wb)
            rparts = R.RefParts(rb, part, k, wb)
            assert O.footprint_proxy(parts) == rparts.footprint_proxy()
            for p in range(k):
                rp_ = rparts.part(p)
                np.testing.assert_array_equal(parts[p].core_nodes, rp_.core_nodes)
                np.testing.assert_array_equal(parts[p].boundary_nodes, rp_.boundary_nodes)
                np.testing.assert_array_equal(parts[p].edges, rp_.edges)
            m = O.materialize(g, parts[k - 1])
            rm = rparts.materialize(k - 1)
            for f in FIELDS:
                np.testing.assert_array_equal(getattr(m, f), rm.field(f), err_msg=f"materialize {f}")


def test_restatement_vs_reference_random_assignments():
    """regrow on random multigraphs with arbitrary (file-style) assignments."""
    R = _ref()
    rng = np.random.default_rng(17)
    for t in range(8):
        ni = int(rng.integers(2, 12))
        na = int(rng.integers(1, 400))
        ands = np.empty((na, 2), np.uint32)
        for q in range(na):
            v = 1 + ni + q
            ands[q] = 2 * rng.integers(0, v, 2) + rng.integers(0, 2, 2)
        outs = (2 * rng.integers(0, 1 + ni + na, 5) + rng.integers(0, 2, 5)).astype(np.uint32)
        raig, rg = R.aig_from_lits(ni, ands, outs)
        g = O.encode(O.Aig(ni, ands, outs, raig.labels))
        for f in FIELDS:
            np.testing.assert_array_equal(getattr(g, f), rg.field(f), err_msg=f)
        k = int(rng.integers(1, 9))
        part = rng.integers(0, k, g.n).astype(np.uint32)
        part[:k] = np.arange(k)
        parts = O.regrow(g, part, k, True)
        rparts = R.RefParts(rg, part, k, True)
        for p in range(k):
            np.testing.assert_array_equal(parts[p].edges, rparts.part(p).edges)
            np.testing.assert_array_equal(parts[p].boundary_nodes, rparts.part(p).boundary_nodes)


@pytest.mark.parametrize("width,copies,seed", [(8, 1, 7), (32, 2, 3), (64, 1, 11)])
def test_restatement_vs_reference_plan_and_forward(width, copies, seed):
    """build_plan arrays bit-exact; fp64 logits of the restated forward (restated
    spmm::execute) vs the shim's forward over the compiled spmm::execute."""
    R = _ref()
    _, rg = R.gen_csa(width)
    rb = R.batch(rg, copies) if copies > 1 else rg
    g = O.batch(O.encode(O.gen_csa(width)), copies) if copies > 1 else O.encode(O.gen_csa(width))
    for thr in ((512, 12, 96), (16, 3, 24)):
        op = O.build_plan(g.row_ptr, *thr)
        rp_ = R.build_plan(g.row_ptr, *thr)
        for key in ("hd_rows", "mid_rows", "ld_groups", "units", "perm"):
            np.testing.assert_array_equal(op[key], rp_[key], err_msg=key)
        O.free_plan(op)
        R.free_plan(rp_)
    prm = O.init_model(seed)
    pred, conf, acc, lg = O.predict_full(g, prm)
    rpred, rconf, racc, rlg = R.predict_full(rb, prm, want_logits=True)
    np.testing.assert_array_equal(lg, rlg)  # same accumulation order end to end
    np.testing.assert_array_equal(pred, rpred)
    np.testing.assert_array_equal(conf, rconf)
    assert acc == racc


def test_partition_lp_restatement_matches_reference_where_it_terminates():
    """the replacement partitioner (oracle restatement of the device
    algorithm) equals the reference's partition_multilevel bit for bit on the
    graphs where the reference terminates and its refined-topo candidate wins."""
    R = _ref()
    for w, k, b in ((64, 2, 1), (64, 4, 1), (32, 3, 4), (128, 2, 1)):
        _, g = R.gen_csa(w)
        if b > 1:
            g = R.batch(g, b)
        rp, ci = g.field("row_ptr"), g.field("col_idx")
        n = rp.shape[0] - 1
        np.testing.assert_array_equal(O.partition_lp(rp, ci, n, k), R.partition_multilevel(g, k, 7))


@pytest.mark.parametrize("w,k", [(64, 8), (64, 16), (32, 64), (16, 7)])
def test_partition_lp_terminates_within_cap(w, k):
    """k >= 8 (the reference livelocks): every part nonempty and within
    ceil(1.05 n / k), deterministic, cut no worse than the topo chunks."""
    g = O.encode(O.gen_csa(w))
    p = O.partition_lp(g.row_ptr, g.col_idx, g.n, k)
    cnt = np.bincount(p, minlength=k)
    assert cnt.min() >= 1 and cnt.max() <= O.lp_cap(g.n, k) and p.max() < k
    np.testing.assert_array_equal(p, O.partition_lp(g.row_ptr, g.col_idx, g.n, k))
    assert O.edge_cut(g, p) <= O.edge_cut(g, O.topo_chunks(g.n, k))
