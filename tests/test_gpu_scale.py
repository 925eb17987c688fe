"""Parity at the BASELINE configurations (BASELINE.json configs 3, 4 and 5).

Every integer stage is compared with the REAL reference code (oracle/_ref,
the reference's own translation units compiled here and shipped prebuilt to
the GPU box), not with the restatement:

  config 5  1024-bit CSA: gen_csa_multiplier (src/circuitgen.cpp:66-133) and
            encode (src/encode.cpp:33-68) of one copy, batch(., 16)
            (src/encode.cpp:70-101) array by array, topo k=64 + regrow
            (src/partition.cpp:301-312, 402-456) of the b16 graph part by part;
            forward logits and classes of one copy (8.4 M rows, i.e. the keyed
            layer-0 + transform-first layer-1 default path the bench runs)
            against predict_full (src/gnn.cpp:293-300: the reference's compiled
            spmm::execute with the restated dense product), then the b16
            classes copy by copy against that verified single copy.
  config 4  512-bit CSA b16: topo k in {2, 4, 8, 64}: part_of, crossing
            fraction, edge cut, every part's core/boundary/edge list, two
            materialized parts; partitioned predict (src/gnn.cpp:280-291) of
            16 regrown k=64 parts (the reference arm's workload) against the
            reference's predict over the same parts.
  config 3  256-bit Booth b8, k=2 regrown: the Booth AIG built through the
            reference's Aig::add_and (src/aig.cpp:10-22) then encode/batch/
            regrow, and predict over both parts.

Bar: bit-exact for the integer stages; logits within LOGIT_RTOL row-normwise;
classes equal on every node whose fp64 top-2 margin exceeds MARGIN_TOL x the
row's max |logit| (near-ties are counted and reported, never hidden).
"""
import os

import numpy as np
import pytest

from helpers import profiled_names, with_env
from oracle import pyoracle as O
from oracle import pyref as R

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

LOGIT_RTOL = 1e-5
MARGIN_TOL = 1e-4
FIELDS = ["row_ptr", "col_idx", "features", "labels", "degree", "fwd_edges"]
MODEL = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "trained_csa8.asg1")


@pytest.fixture(scope="module")
def api():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    if not R.available():
        pytest.skip("oracle/_ref (the compiled reference) is not built")
    from paper_2511_18297_b200 import api as A
    return A


@pytest.fixture(scope="module")
def params():
    return O.load_model(MODEL)[0]


def assert_graph_equal_ref(dev, ref, what):
    """Device graph vs reference graph, one array at a time (bounded host memory)."""
    for f in FIELDS:
        got = dev.copy_out(f)[f]
        exp = ref.field(f)
        assert got.shape == exp.shape, f"{what}: {f} shape {got.shape} != {exp.shape}"
        assert np.array_equal(got, exp), f"{what}: {f} differs at {int(np.argmax(got.ravel() != exp.ravel()))}"
        del got, exp


def assert_parts_equal_ref(dparts, rparts, k, what):
    assert len(dparts) == k
    for p in range(k):
        d, r = dparts[p], rparts.part(p)
        for name in ("core_nodes", "boundary_nodes", "edges"):
            assert np.array_equal(getattr(d, name), getattr(r, name)), f"{what}: part {p} {name}"


def margin_ties(ref_logits):
    s = np.sort(ref_logits, axis=1)
    margin = s[:, -1] - s[:, -2]
    return margin <= MARGIN_TOL * np.maximum(np.abs(ref_logits).max(axis=1), 1e-12)


def check_logits(gpu, ref, what):
    scale = np.maximum(np.abs(ref).max(axis=1), 1e-6)
    err = np.abs(gpu.astype(np.float64) - ref).max(axis=1) / scale
    worst = float(err.max()) if err.size else 0.0
    assert worst <= LOGIT_RTOL, f"{what}: row-normwise logit error {worst:.3e} > {LOGIT_RTOL}"
    return worst


def check_classes(pred, ref_pred, ref_logits, what):
    """Classes equal to the reference's everywhere except at fp64 near-ties."""
    tie = margin_ties(ref_logits)
    diff = pred != ref_pred
    assert not (diff & ~tie).any(), f"{what}: {int((diff & ~tie).sum())} class flips outside near-ties"
    return int(diff.sum()), int(tie.sum())


# ---------------------------------------------------------------------------
# config 5: 1024-bit CSA
# ---------------------------------------------------------------------------
@pytest.fixture(scope="module")
def csa1024(api):
    aig, rg = R.gen_csa(1024)
    c = api.gen_csa_multiplier(1024)
    g = api.encode(c.aig, c.labels)
    return aig, rg, c, g


def test_csa1024_generator_and_encode(api, csa1024):
    aig, rg, c, g = csa1024
    assert c.aig.num_inputs == aig.num_inputs == 2048
    assert np.array_equal(c.aig.and_lits, aig.and_lits)
    assert np.array_equal(c.aig.out_lits, aig.out_lits)
    assert np.array_equal(c.labels, aig.labels)
    assert g.n == 8_381_441
    assert_graph_equal_ref(g, rg, "encode(csa1024)")


def test_csa1024_forward_single_copy(api, csa1024, params):
    """Logits/classes of one 1024-bit copy (8.4 M rows >= 2^20: the keyed layer 0 and
    transform-first layer 1 run, as in the bench) vs the reference predict_full."""
    _, rg, c, g = csa1024
    model = api.Model.from_params(params)
    lg, names = profiled_names(lambda: api.forward(model, g))
    assert "l0_keys" in names and "sage_layer1_xform" in names, names
    rpred, rconf, racc, rlog = R.predict_full(rg, params, want_logits=True)
    worst = check_logits(lg, rlog, "csa1024 b1")
    pred = api.predict_full(model, g)
    flips, ties = check_classes(pred.labels, rpred, rlog, "csa1024 b1 predict_full")
    print(f"csa1024 b1: max logit err {worst:.2e}, {flips} flips at {ties} near-ties, accuracy {pred.accuracy:.6f}")
    if flips == 0:
        assert np.array_equal(pred.confusion, rconf)
        assert pred.accuracy == racc
    # the materialized layer-0 path on the same graph
    lm = with_env("GROOT_L0_KEYED", "0", lambda: api.forward(model, g))
    check_logits(lm, rlog, "csa1024 b1 materialized layer 0")
    # e2e entry point (tile-aligned batch, periodic plan, split last layer) on one copy
    pe = api.classify_aig(model, c.aig, c.labels, copies=1)
    check_classes(pe.labels, rpred, rlog, "csa1024 b1 classify_aig")
    csa1024_ref_cache["pred"], csa1024_ref_cache["logits"] = rpred, rlog
    csa1024_ref_cache["dev_pred"] = pred.labels


csa1024_ref_cache = {}


def test_csa1024_b16_batch_and_classes(api, csa1024, params):
    """batch(g, 16) array by array vs the reference; every copy's classes equal the
    single copy's (verified above against the reference), confusion = 16x."""
    _, rg, c, g = csa1024
    gb = api.batch(g, 16)
    rb = R.batch(rg, 16)
    assert gb.n == 134_103_056 and gb.num_undirected_edges() == 268_107_776
    assert_graph_equal_ref(gb, rb, "batch(csa1024, 16)")
    del rb
    model = api.Model.from_params(params)
    pb = api.predict_full(model, gb)
    p1 = csa1024_ref_cache.get("dev_pred")
    if p1 is None:
        p1 = api.predict_full(model, g).labels
    blocks = pb.labels.reshape(16, -1)
    assert (blocks == p1[None, :]).all(), "a batch copy's classes differ from the single copy's"
    if "pred" in csa1024_ref_cache:
        check_classes(blocks[7], csa1024_ref_cache["pred"], csa1024_ref_cache["logits"], "b16 copy 7")
    single = api.predict_full(model, g)
    assert np.array_equal(pb.confusion, 16 * single.confusion)
    # the e2e call at the bench's configuration: same classes
    pe = api.classify_aig(model, c.aig, c.labels, copies=16)
    assert np.array_equal(pe.labels, pb.labels)
    assert np.array_equal(pe.confusion, pb.confusion)


def test_csa1024_b16_topo64_regrow(api, csa1024):
    """topo k=64 + regrow of the 134 M-node graph vs the reference (its slowest stage)."""
    _, rg, _, g = csa1024
    gb = api.batch(g, 16)
    rb = R.batch(rg, 16)
    k = 64
    pa = api.partition_topo_chunks(gb, k)
    part = R.topo_chunks(rb, k)
    assert np.array_equal(pa.part_of, part)
    assert api.crossing_fraction(gb, pa) == R.crossing_fraction(rb, part, k)
    rparts = R.RefParts(rb, part, k, True)
    dparts = api.regrow(gb, pa)
    assert_parts_equal_ref(dparts, rparts, k, "csa1024 b16 topo64")
    assert api.footprint_proxy(dparts) == rparts.footprint_proxy()
    for p in (0, 37):
        assert_graph_equal_ref(api.materialize(gb, dparts, p), rparts.materialize(p), f"materialize part {p}")


# ---------------------------------------------------------------------------
# config 4: 512-bit CSA b16, partitioned
# ---------------------------------------------------------------------------
@pytest.fixture(scope="module")
def csa512b16(api):
    _, rg = R.gen_csa(512)
    c = api.gen_csa_multiplier(512)
    g = api.encode(c.aig, c.labels)
    gb = api.batch(g, 16)
    rb = R.batch(rg, 16)
    return gb, rb


@pytest.mark.parametrize("k", [2, 4, 8, 64])
def test_csa512_b16_partitions(api, csa512b16, k):
    gb, rb = csa512b16
    pa = api.partition_topo_chunks(gb, k)
    part = R.topo_chunks(rb, k)
    assert np.array_equal(pa.part_of, part)
    cf = api.crossing_fraction(gb, pa)
    assert cf == R.crossing_fraction(rb, part, k)
    assert (cf == 0.0) == (k <= 16), cf  # k | copies: parts are whole copies
    for wb in (True, False):
        rparts = R.RefParts(rb, part, k, wb)
        dparts = api.regrow(gb, pa) if wb else api.core_subgraphs(gb, pa)
        assert_parts_equal_ref(dparts, rparts, k, f"csa512 b16 k={k} regrow={wb}")
        assert api.footprint_proxy(dparts) == rparts.footprint_proxy()
        if wb:
            for p in sorted({0, k // 2 + 1 if k > 2 else 1}):
                assert_graph_equal_ref(api.materialize(gb, dparts, p), rparts.materialize(p),
                                       f"k={k} materialize {p}")


def test_csa512_b16_partitioned_predict(api, csa512b16, params):
    """predict over 16 regrown k=64 parts (straddling copies, with boundary rows) vs the
    reference predict over the same parts: the reference arm's workload shape."""
    gb, rb = csa512b16
    k, first, count = 64, 8, 16
    pa = api.partition_topo_chunks(gb, k)
    dparts = api.regrow(gb, pa)
    rparts = R.RefParts(rb, R.topo_chunks(rb, k), k, True)
    n = gb.n
    rpred = np.zeros(n, np.uint8)
    rlog = np.zeros((n, 5), np.float64)
    R.predict_parts(rparts, first, count, params, pred=rpred, logits=rlog)
    model = api.Model.from_params(params)
    got = api.predict_parts(model, gb, dparts, np.arange(first, first + count))
    core = np.concatenate([dparts[p].core_nodes for p in range(first, first + count)])
    flips, ties = check_classes(got[core], rpred[core], rlog[core], "csa512 b16 k64 predict")
    print(f"csa512 b16 k=64 parts {first}..{first + count - 1}: {core.size} core rows, {flips} flips at {ties} ties")


# ---------------------------------------------------------------------------
# config 3: 256-bit Booth b8, k=2 regrown
# ---------------------------------------------------------------------------
def test_booth256_b8_k2_regrow_predict(api, params):
    c = api.gen_booth_multiplier(256)
    raig, rg = R.aig_from_lits(c.aig.num_inputs, c.aig.and_lits, c.aig.out_lits)
    assert np.array_equal(raig.and_lits, c.aig.and_lits)
    g = api.encode(c.aig, raig.labels)  # the reference's file-style labels (PI/AND/PO)
    assert_graph_equal_ref(g, rg, "encode(booth256)")
    gb = api.batch(g, 8)
    rb = R.batch(rg, 8)
    assert_graph_equal_ref(gb, rb, "batch(booth256, 8)")
    k = 2
    pa = api.partition_topo_chunks(gb, k)
    part = R.topo_chunks(rb, k)
    assert np.array_equal(pa.part_of, part)
    rparts = R.RefParts(rb, part, k, True)
    dparts = api.regrow(gb, pa)
    assert_parts_equal_ref(dparts, rparts, k, "booth256 b8 k2")
    for p in range(k):
        assert_graph_equal_ref(api.materialize(gb, dparts, p), rparts.materialize(p), f"booth materialize {p}")
    n = gb.n
    rpred = np.zeros(n, np.uint8)
    rlog = np.zeros((n, 5), np.float64)
    R.predict_parts(rparts, 0, k, params, pred=rpred, logits=rlog)
    model = api.Model.from_params(params)
    pred = api.predict(model, gb, dparts)
    flips, ties = check_classes(pred.labels, rpred, rlog, "booth256 b8 k2 predict")
    # with no flips the confusion is the reference's over the same labels
    if flips == 0:
        conf = np.zeros((5, 5), np.uint64)
        np.add.at(conf, (rb.field("labels").astype(np.int64), rpred.astype(np.int64)), 1)
        assert np.array_equal(pred.confusion, conf)
    # and the unpartitioned forward of the same graph against predict_full
    fpred, _, _, flog = R.predict_full(rb, params, want_logits=True)
    check_logits(api.forward(model, gb), flog, "booth256 b8 forward")
    check_classes(api.predict_full(model, gb).labels, fpred, flog, "booth256 b8 predict_full")
