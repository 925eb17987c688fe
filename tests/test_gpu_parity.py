"""GPU parity: the CUDA path (through the C ABI) against the oracle and goldens.

Bar: bit-exact for features, CSR, fwd_edges, batch, partition membership,
boundary sets, re-grown edge lists, materialized CSR, plan arrays and classes;
fp32 logits within LOGIT_RTOL of the fp64 oracle, measured row-normwise:
    max_c |gpu - ref| <= LOGIT_RTOL * max(max_c |ref|, 1e-6)
(3xTF32 tensor-core products + fp32 accumulation vs fp64 reference).
Class agreement is required on every node whose fp64 top-2 margin exceeds
MARGIN_TOL * max|logit| of the row; near-ties are counted and reported.
"""
import os

import numpy as np
import pytest

from oracle import pyoracle as O

pytestmark = pytest.mark.gpu

LOGIT_RTOL = 1e-5
MARGIN_TOL = 1e-4
FIELDS = ["row_ptr", "col_idx", "features", "labels", "degree", "fwd_edges"]


@pytest.fixture(scope="module")
def api():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2511_18297_b200 import api as A
    return A


def dev_graph(api, width, copies=1):
    c = api.gen_csa_multiplier(width)
    g = api.encode(c.aig, c.labels)
    return api.batch(g, copies) if copies > 1 else g


def ora_graph(width, copies=1):
    g = O.encode(O.gen_csa(width))
    return O.batch(g, copies) if copies > 1 else g


def assert_graph_equal(dg, hg):
    out = dg.copy_out()
    for f in FIELDS:
        np.testing.assert_array_equal(out[f], getattr(hg, f), err_msg=f)


def check_logits(gpu, ref, what=""):
    gpu = gpu.astype(np.float64)
    scale = np.maximum(np.abs(ref).max(axis=1), 1e-6)
    err = (np.abs(gpu - ref).max(axis=1) / scale)
    worst = float(err.max()) if err.size else 0.0
    assert worst <= LOGIT_RTOL, f"{what}: row-normwise logit error {worst:.3e} > {LOGIT_RTOL}"
    return worst


def check_classes(pred, ref_logits, what=""):
    ref_pred = np.argmax(ref_logits, axis=1)  # first max wins, like Eigen maxCoeff
    s = np.sort(ref_logits, axis=1)
    margin = s[:, -1] - s[:, -2] if ref_logits.shape[1] > 1 else np.full(ref_logits.shape[0], np.inf)
    tie = margin <= MARGIN_TOL * np.maximum(np.abs(ref_logits).max(axis=1), 1e-12)
    bad = (pred != ref_pred) & ~tie
    assert not bad.any(), f"{what}: {int(bad.sum())} class flips outside near-ties"
    return int(((pred != ref_pred) & tie).sum()), int(tie.sum())


# ---------------------------------------------------------------------------
# feature build / CSR / batch
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("width", [2, 3, 8, 16, 64])
def test_encode_bit_exact(api, width):
    assert_graph_equal(dev_graph(api, width), ora_graph(width))


def test_encode_golden(api, golden_dir):
    for w in (2, 8):
        fx = np.load(os.path.join(golden_dir, f"csa{w}.npz"))
        out = dev_graph(api, w).copy_out()
        for f in FIELDS:
            np.testing.assert_array_equal(out[f], fx["g_" + f], err_msg=f)
        out = dev_graph(api, w, 3).copy_out()
        for f in FIELDS:
            np.testing.assert_array_equal(out[f], fx["b3_" + f], err_msg=f)


@pytest.mark.parametrize("width,copies", [(8, 2), (8, 5), (64, 4), (256, 2)])
def test_batch_bit_exact(api, width, copies):
    assert_graph_equal(dev_graph(api, width, copies), ora_graph(width, copies))


def test_encode_parsed_aiger_and_wide_rows(api):
    """AIG with a node of fanout > 4096 (exercises the long-row sort path) and an
    inverted PO driver; parsed from AIGER text."""
    rng = np.random.default_rng(3)
    ni, na = 6, 6000
    ands = np.empty((na, 2), np.uint32)
    for a in range(na):
        v = 1 + ni + a
        ands[a, 0] = 2 * 1 + (a & 1)                      # node 1 drives every AND
        ands[a, 1] = 2 * int(rng.integers(1, v)) + int(rng.integers(0, 2))
    outs = np.array([2 * (ni + na) + 1, 3, 0], np.uint32)
    aig = api.Aig(ni, ands, outs)
    aig2 = api.parse_aiger(api.write_aiger(aig))
    n = aig.num_nodes + outs.shape[0]
    labels = rng.integers(0, 5, n).astype(np.uint8)
    g = api.encode(aig2, labels)
    ref = O.encode(O.Aig(ni, ands, outs, labels))
    assert_graph_equal(g, ref)
    assert int(g.degree[1]) > 4096


def test_graph_from_host_roundtrip(api):
    h = ora_graph(16)
    g = api.EdaGraph.from_host(h.n, h.row_ptr, h.col_idx, h.features, h.labels, h.fwd_edges)
    assert_graph_equal(g, h)
    bad = h.col_idx.copy()
    bad[0] = h.n
    with pytest.raises(ValueError, match="column index out of range"):
        api.EdaGraph.from_host(h.n, h.row_ptr, bad)


# ---------------------------------------------------------------------------
# partition / regrow / materialize
# ---------------------------------------------------------------------------
def assert_parts_equal(dparts, oparts):
    assert len(dparts) == len(oparts)
    for p, op in enumerate(oparts):
        dp = dparts[p]
        np.testing.assert_array_equal(dp.core_nodes, op.core_nodes, err_msg=f"core {p}")
        np.testing.assert_array_equal(dp.boundary_nodes, op.boundary_nodes, err_msg=f"boundary {p}")
        np.testing.assert_array_equal(dp.edges, op.edges, err_msg=f"edges {p}")


@pytest.mark.parametrize("width,copies,k", [(2, 1, 2), (8, 1, 1), (8, 1, 3), (8, 3, 5), (64, 4, 8), (64, 1, 64)])
def test_topo_regrow_materialize_bit_exact(api, width, copies, k):
    g = dev_graph(api, width, copies)
    h = ora_graph(width, copies)
    pa = api.partition_topo_chunks(g, k)
    part = O.topo_chunks(h.n, k)
    np.testing.assert_array_equal(pa.part_of, part)
    assert api.crossing_fraction(g, pa) == O.crossing_fraction(h, part)
    assert api.edge_cut(g, pa) == O.edge_cut(h, part)
    for wb in (True, False):
        dparts = api.regrow(g, pa) if wb else api.core_subgraphs(g, pa)
        oparts = O.regrow(h, part, k, wb)
        assert_parts_equal(dparts, oparts)
        assert api.footprint_proxy(dparts) == O.footprint_proxy(oparts)
        for p in sorted({0, k // 2, k - 1}):
            m = api.materialize(g, dparts, p)
            assert_graph_equal(m, O.materialize(h, oparts[p]))


def test_regrow_golden_and_digests(api, golden_dir):
    fx = np.load(os.path.join(golden_dir, "csa8.npz"))
    g = dev_graph(api, 8)
    for k in (2, 3):
        pa = api.partition_topo_chunks(g, k)
        parts = api.regrow(g, pa)
        for p in range(k):
            key = f"topo{k}_regrow_p{p}_"
            np.testing.assert_array_equal(parts[p].core_nodes, fx[key + "core"])
            np.testing.assert_array_equal(parts[p].boundary_nodes, fx[key + "boundary"])
            np.testing.assert_array_equal(parts[p].edges, fx[key + "edges"])
            m = api.materialize(g, parts, p).copy_out("row_ptr", "col_idx")
            np.testing.assert_array_equal(m["row_ptr"], fx[key + "m_row_ptr"])
            np.testing.assert_array_equal(m["col_idx"], fx[key + "m_col_idx"])


def test_regrow_random_assignments(api):
    """File-style assignments on random multigraphs (duplicates, self loops)."""
    rng = np.random.default_rng(5)
    for t in range(12):
        n = int(rng.integers(2, 3000))
        E = int(rng.integers(0, 4 * n))
        edges = rng.integers(0, n, size=(E, 2)).astype(np.uint32)
        rp, ci = O.build_csr(n, edges)
        h = O.HostGraph(n, rp, ci, rng.integers(0, 2, (n, 4)).astype(np.uint8),
                        rng.integers(0, 5, n).astype(np.uint8), np.diff(rp).astype(np.uint32), edges)
        g = api.EdaGraph.from_host(n, rp, ci, h.features, h.labels, edges)
        k = int(rng.integers(1, min(n, 40) + 1))
        part = rng.integers(0, k, size=n).astype(np.uint32)
        part[:k] = np.arange(k, dtype=np.uint32)  # no empty part
        pa = api.PartitionAssignment.from_host(part)
        assert pa.k == k
        for wb in (True, False):
            dparts = api.regrow(g, pa) if wb else api.core_subgraphs(g, pa)
            oparts = O.regrow(h, part, k, wb)
            assert_parts_equal(dparts, oparts)
        m = api.materialize(g, dparts, k - 1)
        assert_graph_equal(m, O.materialize(h, oparts[k - 1]))


def test_load_assignment_file(api, tmp_path):
    g = dev_graph(api, 8)
    n = g.n
    part = (np.arange(n) * 7 // n).astype(np.uint32)
    path = tmp_path / "assign.txt"
    path.write_text("".join(f"{v} {p}\n" for v, p in enumerate(part.tolist())))
    pa = api.load_assignment(str(path), n)
    np.testing.assert_array_equal(pa.part_of, part)
    assert pa.k == 7
    path.write_text("".join(f"{v} {p}\n" for v, p in enumerate(part.tolist()) if v != 0))
    with pytest.raises(RuntimeError, match="assignment: missing node 0"):
        api.load_assignment(str(path), n)
    with pytest.raises(ValueError, match="k exceeds node count"):
        api.partition_topo_chunks(g, n + 1)


# ---------------------------------------------------------------------------
# row classifier + aggregation
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("width,copies", [(8, 1), (64, 4), (256, 1)])
def test_build_plan_matches_reference(api, width, copies):
    g = dev_graph(api, width, copies)
    h = ora_graph(width, copies)
    for thr in ((512, 12, 96), (64, 4, 32)):
        dp = api.build_plan(g, *thr)
        op = O.build_plan(h.row_ptr, *thr)
        for key in ("perm", "hd_rows", "mid_rows", "ld_groups", "units"):
            np.testing.assert_array_equal(dp[key], op[key], err_msg=key)
        assert (dp["ld_row_begin"], dp["ld_row_end"]) == (op["ld_row_begin"], op["ld_row_end"])
        O.free_plan(op)


@pytest.mark.parametrize("width,copies,f", [(8, 1, 32), (64, 2, 32), (256, 1, 32), (64, 1, 4), (16, 1, 7)])
def test_spmm_mean(api, width, copies, f):
    """LD kernel + HD kernel (PI rows of degree 256 >= threshold at width 256)."""
    g = dev_graph(api, width, copies)
    h = ora_graph(width, copies)
    dense = np.random.default_rng(0xB00B1E5).uniform(-1, 1, size=(h.n, f)).astype(np.float32)
    deg = np.diff(h.row_ptr)
    vals = np.repeat(np.where(deg > 0, 1.0 / np.maximum(deg, 1), 0.0), deg.astype(np.int64))
    plan = O.build_plan(h.row_ptr)
    ref = O.plan_execute(plan, h.row_ptr, h.col_idx, vals, dense.astype(np.float64))
    O.free_plan(plan)
    plan = O.build_plan(h.row_ptr)
    mag = O.plan_execute(plan, h.row_ptr, h.col_idx, vals, np.abs(dense).astype(np.float64))
    O.free_plan(plan)
    out = api.spmm_mean(g, dense)
    # fp32 summation vs fp64: error bounded relative to the operand magnitude D^-1 A |X|
    err = np.abs(out - ref) / np.maximum(mag, 1e-30)
    assert float(err.max()) <= 1e-5, float(err.max())


def test_spmm_csr_identity_and_random(api):
    rng = np.random.default_rng(1)
    n = 1000
    ident = api.spmm_csr(np.arange(n + 1, dtype=np.uint64), np.arange(n, dtype=np.uint32),
                         np.ones(n, np.float32), dense := rng.uniform(-1, 1, (n, 32)).astype(np.float32))
    np.testing.assert_array_equal(ident, dense)
    deg = np.where(rng.random(n) < 0.01, 1024, rng.integers(0, 4, n))
    rp = np.concatenate([[0], np.cumsum(deg)]).astype(np.uint64)
    ci = rng.integers(0, n, int(rp[-1])).astype(np.uint32)
    vals = rng.uniform(-1, 1, int(rp[-1]))
    out = api.spmm_csr(rp, ci, vals.astype(np.float32), dense)
    v64 = vals.astype(np.float32).astype(np.float64)
    ref = O.reference_spmm(rp, ci, v64, dense.astype(np.float64))
    mag = O.reference_spmm(rp, ci, np.abs(v64), np.abs(dense).astype(np.float64))
    assert float((np.abs(out - ref) / np.maximum(mag, 1e-30)).max()) <= 1e-5


# ---------------------------------------------------------------------------
# forward + classify
# ---------------------------------------------------------------------------
def trained_params(golden_dir):
    prm, shape = O.load_model(os.path.join(golden_dir, "trained_csa8.asg1"))
    return prm


@pytest.mark.parametrize("width,copies,seed", [(2, 1, 7), (8, 1, 7), (8, 1, 3), (64, 2, 7), (256, 1, 7)])
def test_forward_logits_and_classes(api, width, copies, seed):
    g = dev_graph(api, width, copies)
    h = ora_graph(width, copies)
    prm = O.init_model(seed)
    model = api.Model.from_params(prm)
    ref = O.forward(h, prm)
    lg = api.forward(model, g)
    check_logits(lg, ref, f"csa{width} b{copies}")
    naive, naive_cls = api.forward_naive(model, g)
    check_logits(naive, ref, "naive path")
    pred = api.predict_full(model, g)
    check_classes(pred.labels, ref, "predict_full")
    opred, oconf, oacc = O.classify(ref, h.labels)
    flips = int((pred.labels != opred).sum())
    assert flips == 0 or flips <= int((np.sort(ref, 1)[:, -1] - np.sort(ref, 1)[:, -2] < 1e-4).sum())
    if flips == 0:
        np.testing.assert_array_equal(pred.confusion, oconf)
        assert pred.accuracy == oacc


def test_forward_trained_model_and_depths(api, golden_dir, tmp_path):
    g = dev_graph(api, 64)
    h = ora_graph(64)
    prm = trained_params(golden_dir)
    model = api.load_model(os.path.join(golden_dir, "trained_csa8.asg1"))
    np.testing.assert_array_equal(model.params, prm)
    ref = O.forward(h, prm)
    check_logits(api.forward(model, g), ref, "trained")
    pred = api.predict_full(model, g)
    check_classes(pred.labels, ref, "trained")
    api.save_model(str(tmp_path / "m.asg1"), model)
    assert open(tmp_path / "m.asg1", "rb").read() == open(os.path.join(golden_dir, "trained_csa8.asg1"), "rb").read()
    for depth in (1, 2, 3, 6):  # BASELINE config 1 names a 3-layer GNN; depth is in the model file
        p = O.init_model(11, depth=depth)
        m = api.Model.from_params(p, depth=depth)
        r = O.forward(h, p, depth=depth)
        check_logits(api.forward(m, g), r, f"depth {depth}")


def test_forward_golden_logits(api, golden_dir):
    for w in (2, 8):
        fx = np.load(os.path.join(golden_dir, f"csa{w}.npz"))
        model = api.Model.from_params(fx["init7_params"])
        g = dev_graph(api, w)
        check_logits(api.forward(model, g), fx["init7_logits"], f"golden csa{w}")
        pred = api.predict_full(model, g)
        check_classes(pred.labels, fx["init7_logits"], f"golden csa{w}")


@pytest.mark.parametrize("width,copies,k", [(8, 1, 1), (8, 1, 4), (64, 2, 8), (64, 1, 16)])
def test_predict_partitioned(api, golden_dir, width, copies, k):
    g = dev_graph(api, width, copies)
    h = ora_graph(width, copies)
    prm = trained_params(golden_dir)
    model = api.Model.from_params(prm)
    pa = api.partition_topo_chunks(g, k)
    for regrown in (True, False):
        parts = api.regrow(g, pa) if regrown else api.core_subgraphs(g, pa)
        pred = api.predict(model, g, parts)
        oparts = O.regrow(h, O.topo_chunks(h.n, k), k, regrown)
        opred, oconf, oacc = O.predict(h, oparts, prm)
        mism = int((pred.labels != opred).sum())
        assert mism == 0, f"k={k} regrow={regrown}: {mism} class mismatches"
        np.testing.assert_array_equal(pred.confusion, oconf)
    if k == 1:  # k=1 regrown partition == whole graph
        np.testing.assert_array_equal(api.predict(model, g, api.regrow(g, pa)).labels,
                                      api.predict_full(model, g).labels)


@pytest.mark.parametrize("circuit,width,copies", [("csa", 32, 3), ("csa", 33, 2), ("csa", 64, 4), ("booth", 16, 3),
                                                   ("csa", 8, 1)])
def test_classify_aig_end_to_end(api, golden_dir, circuit, width, copies):
    """groot_classify_aig (the e2e call): copies go on tile-aligned strides with a
    replicated tile plan when nnz1 % 8 == 0 (else the plain batch); classes and
    confusion come back in the reference's numbering either way."""
    c = (api.gen_booth_multiplier if circuit == "booth" else api.gen_csa_multiplier)(width)
    prm = trained_params(golden_dir)
    model = api.Model.from_params(prm)
    pred = api.classify_aig(model, c.aig, c.labels, copies=copies)
    h1 = O.encode(O.Aig(c.aig.num_inputs, c.aig.and_lits, c.aig.out_lits, c.labels))
    h = O.batch(h1, copies) if copies > 1 else h1
    opred, oconf, oacc, _ = O.predict_full(h, prm)
    np.testing.assert_array_equal(pred.labels, opred)
    np.testing.assert_array_equal(pred.confusion, oconf)


def test_empty_and_edge_cases(api):
    # AIG with inputs only (no ANDs): all rows isolated except PO edges
    aig = api.Aig(3, np.zeros((0, 2), np.uint32), np.array([2, 5], np.uint32))
    g = api.encode(aig)
    ref = O.encode(O.Aig(3, np.zeros((0, 2), np.uint32), np.array([2, 5], np.uint32), np.zeros(6, np.uint8)))
    assert_graph_equal(g, ref)
    prm = O.init_model(7)
    check_logits(api.forward(api.Model.from_params(prm), g), O.forward(ref, prm), "tiny")
    with pytest.raises(ValueError, match="copy count must be >= 1"):
        api.batch(g, 0)
    with pytest.raises(ValueError, match="label count"):
        api.encode(aig, np.zeros(3, np.uint8))


@pytest.mark.slow
def test_large_batch_copy_consistency(api, golden_dir):
    """Size-independent property at a BASELINE size: every batch copy of the
    512-bit b16 graph gets exactly the classes of the single copy, and the
    single copy's classes match the compiled reference's predict_full on every
    node outside fp64 near-ties."""
    from oracle import pyref as R
    prm = trained_params(golden_dir)
    model = api.Model.from_params(prm)
    g1 = dev_graph(api, 512)
    p1 = api.predict_full(model, g1).labels
    _, rg = R.gen_csa(512)
    rpred, _, _, rlog = R.predict_full(rg, prm, want_logits=True)
    check_classes(p1, rlog, "csa512 b1")
    assert ((p1 != rpred) & (p1 != np.argmax(rlog, 1))).sum() == 0
    gb = dev_graph(api, 512, 16)
    assert gb.n == 16 * g1.n
    pb = api.predict_full(model, gb).labels.reshape(16, -1)
    assert (pb == p1[None, :]).all()


def test_shard_device_compute(api, golden_dir):
    """Per-rank device compute of the sharding layer: rank shares computed one
    after another on one GPU and merged equal the single-process reference."""
    from paper_2511_18297_b200 import shard
    prm = trained_params(golden_dir)
    model = api.Model.from_params(prm)
    circ = api.gen_csa_multiplier(16)
    h1 = ora_graph(16)
    compute = shard.device_copy_compute(model, circ)
    world, copies = 3, 5
    blocks, conf = [], np.zeros((5, 5), np.uint64)
    for r in range(world):
        lab, c = compute(shard.copy_shard(r, world, copies, h1.n))
        blocks.append(lab)
        conf += c
    hb = O.batch(h1, copies)
    opred, oconf, _, _ = O.predict_full(hb, prm)
    np.testing.assert_array_equal(np.concatenate(blocks), opred)
    np.testing.assert_array_equal(conf, oconf)
    # partitions: each "rank" forwards only its parts (groot_predict_parts)
    g = dev_graph(api, 16, 2)
    hg = ora_graph(16, 2)
    k = 6
    parts = api.regrow(g, api.partition_topo_chunks(g, k))
    pcompute = shard.device_parts_compute(model, g, parts)
    pred = np.zeros(g.n, np.uint8)
    for r in range(world):
        ids, lab = pcompute(shard.owned_parts(k, r, world))
        pred[ids] = lab
    oparts = O.regrow(hg, O.topo_chunks(hg.n, k), k)
    opred2, _, _ = O.predict(hg, oparts, prm)
    np.testing.assert_array_equal(pred, opred2)


@pytest.mark.parametrize("cap", ["0", "64"])
def test_forward_slow_tiles(api, golden_dir, cap):
    """Tile-plan fallback: with the halo capacity forced down (GROOT_TP_HALO_CAP),
    every tile (cap 0) or the wide-halo tiles (cap 64) gather straight from
    the global CSR; logits and SpMM must still match the oracle."""
    import subprocess
    import sys
    code = f"""
import numpy as np, sys
sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})
from paper_2511_18297_b200 import api
from oracle import pyoracle as O
c = api.gen_csa_multiplier(64); g = api.batch(api.encode(c.aig, c.labels), 2)
h = O.batch(O.encode(O.gen_csa(64)), 2)
prm = O.init_model(7)
lg = api.forward(api.Model.from_params(prm), g)
ref = O.forward(h, prm)
err = (np.abs(lg - ref).max(1) / np.maximum(np.abs(ref).max(1), 1e-6)).max()
assert err <= 1e-5, err
x = np.random.default_rng(3).uniform(-1, 1, (h.n, 32)).astype(np.float32)
out = api.spmm_mean(g, x)
deg = np.diff(h.row_ptr).astype(np.int64)
rows = np.repeat(np.arange(h.n), deg)
s = np.zeros((h.n, 32)); np.add.at(s, rows, x[h.col_idx].astype(np.float64))
ref2 = s / np.maximum(deg, 1)[:, None]
assert np.abs(out - ref2).max() <= 1e-5 * max(1.0, np.abs(ref2).max())
print("ok", err)
"""
    env = dict(os.environ, GROOT_TP_HALO_CAP=cap)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


@pytest.mark.parametrize("width,copies", [(16, 1), (64, 4)])
def test_booth_graph_parity(api, width, copies):
    """BASELINE config 3 family (Booth AIGs): device encode/batch bit-exact vs the
    oracle, topo regrow bit-exact, logits within tolerance, classes match."""
    c = api.gen_booth_multiplier(width)
    g = api.encode(c.aig, c.labels)
    gb = api.batch(g, copies) if copies > 1 else g
    h = O.encode(O.Aig(c.aig.num_inputs, c.aig.and_lits, c.aig.out_lits, c.labels))
    hb = O.batch(h, copies) if copies > 1 else h
    assert_graph_equal(gb, hb)
    k = 3
    parts = api.regrow(gb, api.partition_topo_chunks(gb, k))
    oparts = O.regrow(hb, O.topo_chunks(hb.n, k), k)
    for p in range(k):
        np.testing.assert_array_equal(parts[p].edges, oparts[p].edges)
        np.testing.assert_array_equal(parts[p].boundary_nodes, oparts[p].boundary_nodes)
    prm = O.init_model(7)
    ref = O.forward(hb, prm)
    lg = api.forward(api.Model.from_params(prm), gb)
    check_logits(lg, ref, f"booth{width} b{copies}")
    pred = api.predict_full(api.Model.from_params(prm), gb)
    check_classes(pred.labels, ref, "booth predict_full")


@pytest.mark.parametrize("circuit,width,k", [("csa", 32, 3), ("booth", 16, 4)])
def test_exact_halo_mode_device(api, circuit, width, k):
    """Mode X on the device (groot_layer_dev per rank-local regrown part) with a
    loopback all-to-all between k logical ranks on one GPU: core-row logits
    equal the whole-graph forward of the oracle (predict_full semantics)."""
    import torch
    from paper_2511_18297_b200 import shard
    c = (api.gen_booth_multiplier if circuit == "booth" else api.gen_csa_multiplier)(width)
    g = api.encode(c.aig, c.labels)
    pa = api.partition_topo_chunks(g, k)
    parts = api.regrow(g, pa)
    plans = shard.halo_plans(pa.part_of, [parts[p].core_nodes for p in range(k)],
                             [parts[p].boundary_nodes for p in range(k)])
    prm = O.init_model(7)
    model = api.Model.from_params(prm)
    locs = [api.materialize(g, parts, r) for r in range(k)]
    layers = [shard.device_layer_fn(model, locs[r]) for r in range(k)]
    hs = [None] * k
    for l in range(4):
        hs = [layers[r](l, hs[r]) for r in range(k)]
        if l < 3:
            for r in range(k):
                for q in range(k):
                    if plans[r].send[q].size:
                        src = torch.as_tensor(plans[r].send[q], device="cuda").long()
                        dst = torch.as_tensor(plans[q].recv[r], device="cuda").long()
                        hs[q].index_copy_(0, dst, hs[r].index_select(0, src))
    torch.cuda.synchronize()
    h = O.encode(O.Aig(c.aig.num_inputs, c.aig.and_lits, c.aig.out_lits, c.labels))
    ref = O.forward(h, prm)
    got = np.zeros_like(ref)
    for r in range(k):
        got[parts[r].core_nodes] = hs[r][: plans[r].num_core].cpu().numpy()
    check_logits(got, ref, f"mode X {circuit}{width} k{k}")


def test_encode_rejects_bad_fanins(api):
    """encode's device validation (src/aig.cpp:10-16 semantics): a fanin at or
    above its AND node, or an output driver past the last node, is rejected
    with the reference's message after an in-bounds CSR build; a valid AIG
    encoded right after still matches the oracle."""
    from paper_2511_18297_b200._lib import GrootInvalidArgument
    ands = np.array([[2, 4], [6, 12]], np.uint32)  # node 4 = AND(1, 2); node 5 = AND(3, node 6: forward reference)
    with pytest.raises(GrootInvalidArgument, match="fanin index must be strictly below the new node"):
        api.encode(api.Aig(3, ands, np.array([10], np.uint32)))
    ands_ok = np.array([[2, 4], [6, 8]], np.uint32)
    with pytest.raises(GrootInvalidArgument, match="driver references unknown node"):
        api.encode(api.Aig(3, ands_ok, np.array([40], np.uint32)))  # output driver 20 > last node
    c = api.gen_csa_multiplier(8)
    got = api.encode(c.aig, c.labels).copy_out()
    ref = O.encode(O.gen_csa(8))
    for f in ("row_ptr", "col_idx", "features", "fwd_edges"):
        assert np.array_equal(got[f], getattr(ref, f)), f


@pytest.mark.parametrize("width,copies,trained", [(64, 2, True), (256, 1, False), (64, 1, False)])
def test_certified_head(api, golden_dir, width, copies, trained):
    """Last layer without logits (GROOT_HEAD_CERT): classes from the single-operand
    tensor-core head where its margin bound certifies them, the exact fp32 head
    elsewhere. Default, all-exact (bound scale 1e30) and the oracle must agree
    off fp64 near-ties; with logits requested every row takes the exact head."""
    from helpers import near_ties, with_env
    g = dev_graph(api, width, copies)
    h = ora_graph(width, copies)
    prm = trained_params(golden_dir) if trained else O.init_model(5)
    model = api.Model.from_params(prm)
    ref = O.forward(h, prm)
    dflt = api.predict_full(model, g)
    exact = with_env("GROOT_HEAD_CERT_SCALE", "1e30", lambda: api.predict_full(model, g))
    check_classes(dflt.labels, ref, "certified head")
    check_classes(exact.labels, ref, "exact head")
    assert_same = (dflt.labels != exact.labels) & ~near_ties(ref)
    assert not assert_same.any()
    check_logits(api.forward(model, g), ref, "logits (exact head)")


def test_certified_head_ties_take_first_max(api):
    """Two identical class columns: their logits tie exactly, the margin test
    fails, the exact head keeps the first maximum (class 0, never class 1),
    as Eigen's maxCoeff in the reference (src/gnn.cpp:293-300)."""
    g = dev_graph(api, 64, 2)
    h = ora_graph(64, 2)
    prm = O.init_model(7).copy()
    wo = prm.shape[0] - (32 * 5 + 5)
    W = prm[wo:wo + 160].reshape(32, 5)
    W[:, 1] = W[:, 0]
    prm[wo + 160 + 1] = prm[wo + 160]
    model = api.Model.from_params(prm)
    ref = O.forward(h, prm)
    pred = api.predict_full(model, g)
    from helpers import near_ties
    assert not (pred.labels == 1).any()
    check_classes(pred.labels, ref, "tied columns")
    sure = (np.argmax(ref, axis=1) == 0) & ~near_ties(np.delete(ref, 1, axis=1))
    assert sure.sum() > 0
    assert (pred.labels[sure] == 0).all()
