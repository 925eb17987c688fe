"""Device partition_multilevel replacement (csrc/partition_lp.cu).

Bit-exact against the oracle restatement (oracle/pyoracle.py:partition_lp) on
CSA / Booth / random graphs, including HD rows (CTA path, histogram and
quadratic variants), and against the compiled reference's
partition_multilevel (src/partition.cpp:314-367) where that terminates. At
k >= 8 (reference livelock) and at BASELINE size: within the 5 % cap, no empty
part, deterministic, and the result feeds regrow / predict.
"""
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


def check_props(part, n, k):
    cnt = np.bincount(part, minlength=k)
    assert part.max() < k and cnt.min() >= 1 and cnt.max() <= O.lp_cap(n, k)


@pytest.mark.parametrize("circuit,width,copies,k", [
    ("csa", 64, 1, 2), ("csa", 64, 1, 3), ("csa", 64, 1, 8), ("csa", 64, 1, 64), ("csa", 32, 4, 3),
    ("csa", 256, 1, 16), ("csa", 256, 1, 10000), ("booth", 64, 2, 8), ("csa", 8, 1, 457), ("csa", 8, 1, 1)])
def test_device_equals_oracle(api, circuit, width, copies, k):
    c = (api.gen_booth_multiplier if circuit == "booth" else api.gen_csa_multiplier)(width)
    g = api.encode(c.aig, c.labels)
    if copies > 1:
        g = api.batch(g, copies)
    h = g.copy_out("row_ptr", "col_idx")
    n = g.n
    stats = {}
    pa = api.partition_multilevel(g, k, 7, stats)
    exp = O.partition_lp(h["row_ptr"], h["col_idx"], n, k)
    np.testing.assert_array_equal(pa.part_of, exp)
    assert pa.k == k
    check_props(pa.part_of, n, k)
    np.testing.assert_array_equal(api.partition_multilevel(g, k, 3).part_of, exp)  # deterministic, any seed
    if 1 < k < n:
        assert api.edge_cut(g, pa) <= api.edge_cut(g, api.partition_topo_chunks(g, k))


def test_random_graphs_with_hd_rows(api):
    rng = np.random.default_rng(21)
    for t in range(6):
        n = int(rng.integers(300, 4000))
        e = [(int(u), v) for v in range(1, n) for u in rng.integers(0, v, rng.integers(1, 5))]
        hub = int(rng.integers(0, n))
        e += [(hub, int(v)) for v in rng.choice(n, 300, replace=False) if v != hub]  # one HD row
        e = np.array(e, np.uint32)
        rp, ci = O.build_csr(n, e)
        g = api.EdaGraph.from_host(n, rp, ci, None, None, e)
        for k in (2, 5, 13):
            pa = api.partition_multilevel(g, k)
            np.testing.assert_array_equal(pa.part_of, O.partition_lp(rp, ci, n, k))
            check_props(pa.part_of, n, k)


def test_equals_reference_where_it_terminates(api):
    from oracle import pyref as R
    if not R.available():
        pytest.skip("oracle/_ref not built")
    for w, k in ((64, 2), (64, 4), (128, 2)):
        c = api.gen_csa_multiplier(w)
        g = api.encode(c.aig, c.labels)
        _, rg = R.gen_csa(w)
        np.testing.assert_array_equal(api.partition_multilevel(g, k).part_of, R.partition_multilevel(rg, k, 7))


def test_errors(api):
    c = api.gen_csa_multiplier(4)
    g = api.encode(c.aig, c.labels)
    with pytest.raises(ValueError, match="k exceeds node count"):
        api.partition_multilevel(g, g.n + 1)
    with pytest.raises(ValueError, match="k must be >= 1"):
        api.partition_multilevel(g, 0)


@pytest.mark.slow
def test_baseline_size_straddling_cut(api, golden_dir):
    """1024-bit CSA b1 into 8 parts (config 5's copy over 8 GPUs): parts straddle the
    copy, within the cap; regrow + predict over them run; the cut is far below topo's."""
    import os
    import time
    c = api.gen_csa_multiplier(1024)
    g = api.encode(c.aig, c.labels)
    k = 8
    t0 = time.perf_counter()
    stats = {}
    pa = api.partition_multilevel(g, k, 7, stats)
    dt = time.perf_counter() - t0
    part = pa.part_of
    check_props(part, g.n, k)
    cut, tcut = api.edge_cut(g, pa), api.edge_cut(g, api.partition_topo_chunks(g, k))
    print(f"csa1024 k=8: cut {cut} vs topo {tcut}, {stats}, {dt * 1e3:.1f} ms")
    assert 0 < cut < tcut
    model = api.load_model(os.path.join(golden_dir, "trained_csa8.asg1"))
    pred = api.predict(model, g, api.regrow(g, pa))
    assert pred.labels.shape[0] == g.n and 0.5 < pred.accuracy <= 1.0
