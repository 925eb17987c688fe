"""Boundary completion (round 2) on the device, through the C ABI.

* SageContext / make_context (src/gnn.cpp:140-178): forward(model, ctx) equals
  forward(model, g); release + rebuild gives the same logits.
* predict(model, g, parts) consumes the parts it is given (groot_parts_from_host),
  including hand-made parts the reference would accept.
* spmm: degree_sort / build_plan over a host row_ptr (src/spmm.cpp:9-127), and
  execute over CsrMatrix<double> bit for bit (inc/spmm.hpp:106-225).
* arbitrary u8 features (not just 0/1) in the materialized layer 0;
  regrow / crossing_fraction / edge_cut refuse a CSR-only graph.
"""
import os

import numpy as np
import pytest

from oracle import pyoracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2511_18297_b200 import api as A
    return A


def rel_err(a, ref):
    return float((np.abs(a.astype(np.float64) - ref).max(1) / np.maximum(np.abs(ref).max(1), 1e-6)).max())


def test_make_context_forward(api):
    c = api.gen_csa_multiplier(64)
    g = api.batch(api.encode(c.aig, c.labels), 3)
    prm = O.init_model(7)
    model = api.Model.from_params(prm)
    ctx = api.make_context(g)
    a = api.forward(model, ctx)
    b = api.forward(model, g)
    np.testing.assert_array_equal(a, b)
    ctx.release()
    np.testing.assert_array_equal(api.forward(model, g), a)  # rebuilt on demand
    h = O.batch(O.encode(O.gen_csa(64)), 3)
    assert rel_err(a, O.forward(h, prm)) <= 1e-5
    p = api.predict_full(model, api.make_context(g))
    assert np.array_equal(p.labels, api.predict_full(model, g).labels)
    np.testing.assert_array_equal(ctx.labels, h.labels)


def test_predict_consumes_given_parts(api, golden_dir):
    prm = O.load_model(os.path.join(golden_dir, "trained_csa8.asg1"))[0]
    model = api.Model.from_params(prm)
    c = api.gen_csa_multiplier(32)
    g = api.batch(api.encode(c.aig, c.labels), 2)
    h = O.batch(O.encode(O.gen_csa(32)), 2)
    k = 5
    oparts = O.regrow(h, O.topo_chunks(h.n, k), k)
    host_parts = [api.AugmentedPartition(p.core_nodes, p.boundary_nodes, p.edges) for p in oparts]
    got = api.predict(model, g, host_parts)
    exp, econf, eacc = O.predict(h, oparts, prm)
    np.testing.assert_array_equal(got.labels, exp)
    np.testing.assert_array_equal(got.confusion, econf)
    # hand-made parts: part 0's boundary dropped -- a different prediction, but
    # the one the reference computes for exactly these parts
    cut = [O.Part(oparts[0].core_nodes, np.zeros(0, np.uint32),
                  oparts[0].edges[(oparts[0].edges < oparts[0].core_nodes.size).all(1)])] + list(oparts[1:])
    got2 = api.predict(model, g, [api.AugmentedPartition(p.core_nodes, p.boundary_nodes, p.edges) for p in cut])
    exp2, _, _ = O.predict(h, cut, prm)
    np.testing.assert_array_equal(got2.labels, exp2)


def test_degree_sort_and_plan_from_row_ptr(api):
    h = O.batch(O.encode(O.gen_csa(64)), 2)
    perm, srp = api.degree_sort(h.row_ptr)
    operm, osrp = O.degree_sort(h.row_ptr)
    np.testing.assert_array_equal(perm, operm)
    np.testing.assert_array_equal(srp, osrp)
    for thr in ((512, 12, 96), (64, 4, 32)):
        dp = api.build_plan_rows(h.row_ptr, *thr)
        op = O.build_plan(h.row_ptr, *thr)
        for key in ("perm", "hd_rows", "mid_rows", "ld_groups", "units"):
            np.testing.assert_array_equal(dp[key], op[key], err_msg=key)
        O.free_plan(op)
    with pytest.raises(ValueError, match="hd_threshold must exceed ld_threshold"):
        api.build_plan_rows(h.row_ptr, 4, 12, 96)


def test_spmm_f64_bitwise(api):
    rng = np.random.default_rng(4)
    n = 3000
    deg = np.where(rng.random(n) < 0.01, 700, rng.integers(0, 6, n))
    rp = np.concatenate([[0], np.cumsum(deg)]).astype(np.uint64)
    ci = rng.integers(0, n, int(rp[-1])).astype(np.uint32)
    vals = rng.uniform(-1, 1, int(rp[-1]))
    dense = rng.uniform(-1, 1, (n, 32))
    out0 = api.spmm_csr_f64(rp, ci, vals, dense, hd_threshold=0)
    np.testing.assert_array_equal(out0, O.reference_spmm(rp, ci, vals, dense))  # reference_spmm, bit for bit
    for hd in (512, 64):
        plan = O.build_plan(rp, hd, 12 if hd > 12 else 4, 96)
        ex = O.plan_execute(plan, rp, ci, vals, dense)
        O.free_plan(plan)
        np.testing.assert_array_equal(api.spmm_csr_f64(rp, ci, vals, dense, hd_threshold=hd), ex)  # execute, bit for bit
    # float: the same order in fp32
    out32 = api.spmm_csr(rp, ci, vals.astype(np.float32), dense.astype(np.float32), hd_threshold=0)
    ref32 = np.zeros_like(out32)
    for r in range(n):
        acc = np.zeros(32, np.float32)
        for q in range(int(rp[r]), int(rp[r + 1])):
            acc = acc + np.float32(vals[q]) * dense[ci[q]].astype(np.float32)
        ref32[r] = acc
    np.testing.assert_array_equal(out32, ref32)


def test_layer0_non_binary_features(api):
    """Feature values up to 255 with degrees >= 2: the packed byte counters would
    carry into the next feature; the layer must count per feature."""
    rng = np.random.default_rng(8)
    n = 4000
    e = []
    for v in range(1, n):
        for u in rng.integers(0, v, rng.integers(1, 12)):
            e.append((int(u), v))
    e = np.array(e, np.uint32)
    rp, ci = O.build_csr(n, e)
    for hi in (2, 3, 255):
        feat = rng.integers(0, hi + 1, (n, 4)).astype(np.uint8)
        feat[::5] = 255
        g = api.EdaGraph.from_host(n, rp, ci, feat, np.zeros(n, np.uint8), e)
        hg = O.HostGraph(n, rp, ci, feat, np.zeros(n, np.uint8), np.diff(rp).astype(np.uint32), e)
        for depth in (1, 2, 4):
            prm = O.init_model(9, depth=depth)
            lg = api.forward(api.Model.from_params(prm, depth=depth), g)
            assert rel_err(lg, O.forward(hg, prm, depth=depth)) <= 1e-5, (hi, depth)


def test_csr_only_graph_refuses_edge_walks(api):
    h = O.encode(O.gen_csa(8))
    g = api.EdaGraph.from_host(h.n, h.row_ptr, h.col_idx, h.features, h.labels)  # no fwd_edges
    pa = api.partition_topo_chunks(g, 2)
    for fn in (lambda: api.regrow(g, pa), lambda: api.crossing_fraction(g, pa), lambda: api.edge_cut(g, pa)):
        with pytest.raises(ValueError, match="fwd_edges required"):
            fn()


def test_per_device_stream_roundtrip(api):
    """groot_set_stream is per device: setting and reading back on device 0."""
    import torch
    from paper_2511_18297_b200 import _lib
    L = _lib.lib()
    s = torch.cuda.Stream()
    old = L.groot_get_stream()
    assert L.groot_set_stream(s.cuda_stream) == 0
    assert L.groot_get_stream() == s.cuda_stream
    c = api.gen_csa_multiplier(16)
    g = api.encode(c.aig, c.labels)
    prm = O.init_model(3)
    lg = api.forward(api.Model.from_params(prm), g)
    assert rel_err(lg, O.forward(O.encode(O.gen_csa(16)), prm)) <= 1e-5
    assert L.groot_set_stream(old) == 0
