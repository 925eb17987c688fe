"""Keyed layer 0 (forward.cu, l0_key_kernel / dict_finalize_kernel): layer 1
reads entry rows of a record dictionary instead of materialized layer-0 rows.

The entry rows are computed with the layer-0 kernel's own arithmetic, so with
layer 1 on the tensor cores (GROOT_L1_XFORM=0, and always when layer 1 is the
last layer) the keyed forward is BIT-identical to the materialized one
(GROOT_L0_KEYED=0). By default a keyed layer 1 followed by more layers runs
transform-first (kModeXform: entry rows . W once, then a gather-sum of the
transformed rows): a different but exact-in-reals evaluation order, held to
5e-6 of the materialized forward and to the oracle's 1e-5. Graphs that are not
keyable (non-binary features, more than 255 distinct records) must fall back
to the materialized path and still match the oracle.
"""
import os

import numpy as np
import pytest

from helpers import assert_same_classes_off_ties, profiled_names, rel_err, with_env
from oracle import pyoracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2511_18297_b200 import api as A
    return A


@pytest.fixture(autouse=True)
def keyed_on_small_graphs():
    """The library keys only graphs of >= 2^20 rows by default; these tests use small ones."""
    old = os.environ.get("GROOT_L0_KEYED_MIN_ROWS")
    os.environ["GROOT_L0_KEYED_MIN_ROWS"] = "0"
    yield
    if old is None:
        del os.environ["GROOT_L0_KEYED_MIN_ROWS"]
    else:
        os.environ["GROOT_L0_KEYED_MIN_ROWS"] = old


@pytest.mark.parametrize("circuit,width,copies,depth", [("csa", 64, 2, 4), ("csa", 256, 1, 2), ("booth", 16, 3, 3),
                                                        ("csa", 8, 1, 4)])
def test_keyed_bit_identical_to_materialized(api, circuit, width, copies, depth):
    c = api.gen_csa_multiplier(width) if circuit == "csa" else api.gen_booth_multiplier(width)
    g = api.encode(c.aig, c.labels)
    if copies > 1:
        g = api.batch(g, copies)
    prm = O.init_model(5, depth=depth)
    model = api.Model.from_params(prm, depth=depth)
    keyed, names = profiled_names(lambda: api.forward(model, g))
    assert "l0_keys" in names and "sage_layer0" not in names, names
    assert ("sage_layer1_xform" in names) == (depth > 2), names
    plain = with_env("GROOT_L0_KEYED", "0", lambda: api.forward(model, g))
    keyed_mma = with_env("GROOT_L1_XFORM", "0", lambda: api.forward(model, g))
    np.testing.assert_array_equal(keyed_mma, plain)  # same arithmetic as the materialized path
    if depth == 2:
        np.testing.assert_array_equal(keyed, plain)
    assert rel_err(keyed, plain.astype(np.float64)) <= 5e-6
    h = O.encode(O.Aig(c.aig.num_inputs, c.aig.and_lits, c.aig.out_lits, c.labels))
    if copies > 1:
        h = O.batch(h, copies)
    ref = O.forward(h, prm, depth=depth)
    assert rel_err(keyed, ref) <= 1e-5
    p1 = api.predict_full(model, g)
    s2 = np.sort(ref, 1)
    tie = (s2[:, -1] - s2[:, -2]) <= 1e-4 * np.maximum(np.abs(ref).max(1), 1e-12)
    assert not ((p1.labels != np.argmax(ref, 1)) & ~tie).any()


def test_keyed_classify_aig_matches_materialized(api, golden_dir):
    """groot_classify_aig (tile-aligned batch, periodic plan, split last layer)."""
    model = api.load_model(os.path.join(golden_dir, "trained_csa8.asg1"))
    c = api.gen_csa_multiplier(64)
    r1 = with_env("GROOT_L1_XFORM", "0", lambda: api.classify_aig(model, c.aig, c.labels, 5))
    r0 = with_env("GROOT_L0_KEYED", "0", lambda: api.classify_aig(model, c.aig, c.labels, 5))
    np.testing.assert_array_equal(r1.labels, r0.labels)
    np.testing.assert_array_equal(r1.confusion, r0.confusion)
    rx = api.classify_aig(model, c.aig, c.labels, 5)  # default: transform-first layer 1
    h = O.batch(O.encode(O.Aig(c.aig.num_inputs, c.aig.and_lits, c.aig.out_lits, c.labels)), 5)
    ref = O.forward(h, O.load_model(os.path.join(golden_dir, "trained_csa8.asg1"))[0])
    # transform-first vs materialized: fp32 rounding differs, so labels may differ
    # only where the fp64 reference itself is a near-tie
    assert_same_classes_off_ties(rx.labels, r0.labels, ref, "transform-first vs materialized")
    assert_same_classes_off_ties(rx.labels, np.argmax(ref, 1), ref, "transform-first vs oracle")


def random_graph(n, max_deg, seed, feat_max=1):
    rng = np.random.default_rng(seed)
    e = []
    for v in range(1, n):
        for u in rng.integers(0, v, rng.integers(1, max_deg)):
            e.append((int(u), v))
    e = np.array(e, np.uint32)
    rp, ci = O.build_csr(n, e)
    feat = rng.integers(0, feat_max + 1, (n, 4)).astype(np.uint8)
    return rp, ci, feat


@pytest.mark.parametrize("case", ["non_binary", "many_records", "keyable_random"])
def test_keyed_fallback(api, case):
    if case == "non_binary":
        rp, ci, feat = random_graph(3000, 6, 1, feat_max=2)
    elif case == "many_records":  # ~2100 distinct records
        rp, ci, feat = random_graph(3000, 3, 3)
    else:  # sparse binary features: ~90 distinct records
        rp, ci, feat = random_graph(3000, 3, 3)
        feat[:] = 0
        feat[::7, 0] = 1
    n = feat.shape[0]
    g = api.EdaGraph.from_host(n, rp, ci, feat, np.zeros(n, np.uint8))
    prm = O.init_model(9)
    model = api.Model.from_params(prm)
    lg, names = profiled_names(lambda: api.forward(model, g))
    h = O.HostGraph(n, rp, ci, feat, np.zeros(n, np.uint8), np.diff(rp).astype(np.uint32), np.zeros((0, 2), np.uint32))
    assert rel_err(lg, O.forward(h, prm)) <= 1e-5
    keyed = case == "keyable_random"
    assert ("sage_layer0" in names) != keyed, names
    if keyed:
        plain = with_env("GROOT_L0_KEYED", "0", lambda: api.forward(model, g))
        np.testing.assert_array_equal(with_env("GROOT_L1_XFORM", "0", lambda: api.forward(model, g)), plain)
        assert rel_err(lg, plain.astype(np.float64)) <= 5e-6


@pytest.mark.parametrize("cap", ["0", "64"])
def test_keyed_slow_tiles(cap):
    """Keyed + transform-first layers with the tile plan's fallback forced
    (GROOT_TP_HALO_CAP): slow tiles gather entry rows from global memory."""
    import subprocess
    import sys
    code = f"""
import numpy as np, sys
sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})
from paper_2511_18297_b200 import api
from oracle import pyoracle as O
c = api.gen_csa_multiplier(64); g = api.batch(api.encode(c.aig, c.labels), 2)
h = O.batch(O.encode(O.gen_csa(64)), 2)
for depth in (2, 4):
    prm = O.init_model(3, depth=depth)
    lg = api.forward(api.Model.from_params(prm, depth=depth), g)
    ref = O.forward(h, prm, depth=depth)
    err = (np.abs(lg - ref).max(1) / np.maximum(np.abs(ref).max(1), 1e-6)).max()
    assert err <= 1e-5, (depth, err)
print("ok")
"""
    env = dict(os.environ, GROOT_TP_HALO_CAP=cap, GROOT_L0_KEYED_MIN_ROWS="0")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


@pytest.mark.parametrize("circuit,width,copies,depth", [("booth", 64, 2, 4), ("csa", 160, 1, 6)])
def test_keyed_more_shapes(api, circuit, width, copies, depth):
    """Booth (more record kinds) and a deep model (transform-first layer 1 then four tensor-core layers),
    HD rows included (CSA 160: PI degree 160)."""
    c = api.gen_csa_multiplier(width) if circuit == "csa" else api.gen_booth_multiplier(width)
    g = api.encode(c.aig, c.labels)
    if copies > 1:
        g = api.batch(g, copies)
    prm = O.init_model(13, depth=depth)
    model = api.Model.from_params(prm, depth=depth)
    lg, names = profiled_names(lambda: api.forward(model, g))
    h = O.encode(O.Aig(c.aig.num_inputs, c.aig.and_lits, c.aig.out_lits, c.labels))
    if copies > 1:
        h = O.batch(h, copies)
    ref = O.forward(h, prm, depth=depth)
    assert rel_err(lg, ref) <= 1e-5
    if "l0_keys" in names and "sage_layer0" not in names:
        assert "sage_layer1_xform" in names
    r1 = api.classify_aig(model, c.aig, c.labels, 3)
    r0 = with_env("GROOT_L0_KEYED", "0", lambda: api.classify_aig(model, c.aig, c.labels, 3))
    ref3 = np.tile(ref if copies == 1 else ref[: ref.shape[0] // copies], (3, 1))
    assert_same_classes_off_ties(r1.labels, r0.labels, ref3, "keyed vs materialized classify_aig")
    assert_same_classes_off_ties(r1.labels, np.argmax(ref3, 1), ref3, "keyed classify_aig vs oracle")


def test_small_graphs_stay_materialized(api):
    """Below GROOT_L0_KEYED_MIN_ROWS (default 2^20 rows) the key passes' launch cost
    exceeds what they save: layer 0 is materialized."""
    c = api.gen_csa_multiplier(16)
    g = api.encode(c.aig, c.labels)
    model = api.Model.from_params(O.init_model(2))
    del os.environ["GROOT_L0_KEYED_MIN_ROWS"]  # the library default (restored by the fixture)
    try:
        _, names = profiled_names(lambda: api.forward(model, g))
    finally:
        os.environ["GROOT_L0_KEYED_MIN_ROWS"] = "0"
    assert "sage_layer0" in names and "l0_keys" not in names, names


def local_graph(n, max_fanin, window, seed):
    """Neighbours within `window` rows (tiles stay under the staged-halo cap, so
    the tile kernels take the row-record path), degrees well above the four
    slots a row record holds inline."""
    rng = np.random.default_rng(seed)
    e = []
    for v in range(1, n):
        lo = max(0, v - window)
        for u in rng.integers(lo, v, rng.integers(1, max_fanin)):
            e.append((int(u), v))
    rp, ci = O.build_csr(n, np.array(e, np.uint32))
    feat = (rng.random((n, 4)) < 0.5).astype(np.uint8)
    return rp, ci, feat


@pytest.mark.parametrize("seed,sparse", [(11, True), (12, True), (13, False)])
def test_row_records_long_rows(api, seed, sparse):
    """Rows of degree > 4 finish their neighbour sums from the staged slot list
    (tile_plan.cuh row records hold four slots inline): forwards against the
    oracle on graphs where most rows are that long. Sparse features: keyed
    (and its tensor-core variant bit-identical to the materialized forward);
    dense features: not keyable, the materialized path."""
    rp, ci, feat = local_graph(4000, 7, 60, seed)  # no slow tiles, ~80 % of rows longer than 4
    if sparse:
        feat[:] = 0
        feat[::13, 0] = 1
    deg = np.diff(rp)
    assert (deg > 4).mean() > 0.5 and deg.max() < 128
    n = feat.shape[0]
    g = api.EdaGraph.from_host(n, rp, ci, feat, np.zeros(n, np.uint8))
    prm = O.init_model(seed)
    model = api.Model.from_params(prm)
    h = O.HostGraph(n, rp, ci, feat, np.zeros(n, np.uint8), deg.astype(np.uint32), np.zeros((0, 2), np.uint32))
    ref = O.forward(h, prm)
    lg, names = profiled_names(lambda: api.forward(model, g))
    assert ("sage_layer0" not in names) == sparse, names
    assert rel_err(lg, ref) <= 1e-5
    assert_same_classes_off_ties(np.argmax(lg, 1), np.argmax(ref, 1), ref, "forward vs oracle")
    if sparse:
        plain = with_env("GROOT_L0_KEYED", "0", lambda: api.forward(model, g))
        assert rel_err(plain, ref) <= 1e-5
        np.testing.assert_array_equal(with_env("GROOT_L1_XFORM", "0", lambda: api.forward(model, g)), plain)


@pytest.mark.parametrize("threshold", ["256", "16"])
def test_row_records_hd_threshold(threshold):
    """Row records under other row-classifier thresholds (GROOT_HD_THRESHOLD,
    read once per process): 256 makes rows of degree 128..255 LD rows (their
    degree needs the record's eighth degree bit), 16 makes rows of degree >= 16
    HD rows. Keyed (sparse features) and materialized forwards vs the oracle."""
    import subprocess
    import sys
    code = f"""
import numpy as np, sys
sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})
from paper_2511_18297_b200 import api
from oracle import pyoracle as O
rng = np.random.default_rng(5)
n = 5000
e = [(int(u), v) for v in range(1, n) for u in rng.integers(max(0, v - 40), v, rng.integers(1, 4))]
for hub in range(10, n - 128, 640):  # a few rows of degree ~190 with in-tile neighbours (repeated edges)
    e += [(hub, int(v)) for v in rng.integers(hub + 1, hub + 110, 190)]
rp, ci = O.build_csr(n, np.array(e, np.uint32))
deg = np.diff(rp.astype(np.int64))
assert deg.max() >= 150 and deg.max() < 256, deg.max()
for sparse in (True, False):
    feat = (rng.random((n, 4)) < 0.5).astype(np.uint8)
    if sparse:
        feat[:] = 0
        feat[::11, 1] = 1
    g = api.EdaGraph.from_host(n, rp, ci, feat, np.zeros(n, np.uint8))
    prm = O.init_model(4)
    lg = api.forward(api.Model.from_params(prm), g)
    h = O.HostGraph(n, rp, ci, feat, np.zeros(n, np.uint8), deg.astype(np.uint32), np.zeros((0, 2), np.uint32))
    ref = O.forward(h, prm)
    err = (np.abs(lg - ref).max(1) / np.maximum(np.abs(ref).max(1), 1e-6)).max()
    assert err <= 1e-5, (sparse, err)
print("ok")
"""
    env = dict(os.environ, GROOT_HD_THRESHOLD=threshold, GROOT_L0_KEYED_MIN_ROWS="0")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
