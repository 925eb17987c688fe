"""Verification consumer of the classes: backward_rewrite
(src/verify.cpp:220-395, restated Boost-free in csrc/verify.cpp), host code.

The reference verifier needs Boost.Multiprecision (absent), so it cannot run
here; its verdicts are pinned instead by exhaustive simulation
(truth_table_equiv, simulate) and by known answers: a correct multiplier is
equivalent with any labels (labels only guide, wrong ones cost time), a
mutated one never is.
"""
import numpy as np
import pytest

from paper_2511_18297_b200 import api


@pytest.mark.parametrize("width", [2, 3, 4, 6, 8, 12, 16, 32])
def test_ground_truth_labels_prove_csa(width):
    c = api.gen_csa_multiplier(width)
    r = api.backward_rewrite(c.aig, c.labels, width, c.supports)
    assert r.equivalent and not r.inconclusive and r.residual_terms == 0 and r.residual == ""
    # every half / full adder collapses through the XOR/MAJ shortcut with supports given
    assert r.shortcut_count == width * (width - 1) and r.fallback_count == 0
    r2 = api.backward_rewrite(c.aig, c.labels, width)  # structural supports only
    assert r2.equivalent and r2.fallback_count == 0
    if width <= 8:
        assert api.truth_table_equiv(c.aig, width)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_wrong_labels_are_never_unsound(seed):
    rng = np.random.default_rng(seed)
    w = 5
    c = api.gen_csa_multiplier(w)
    labels = rng.integers(0, 5, c.labels.shape[0]).astype(np.uint8)
    r = api.backward_rewrite(c.aig, labels, w)
    assert r.equivalent or r.inconclusive


@pytest.mark.parametrize("mutation", ["fanin", "output", "swap"])
def test_mutated_multiplier_is_refuted(mutation):
    w = 6
    c = api.gen_csa_multiplier(w)
    ands, outs = c.aig.and_lits.copy(), c.aig.out_lits.copy()
    if mutation == "fanin":
        ands[ands.shape[0] // 3, 1] ^= 1
    elif mutation == "output":
        outs[5] ^= 1
    else:
        outs[[2, 3]] = outs[[3, 2]]
    bad = api.Aig(c.aig.num_inputs, ands, outs)
    r = api.backward_rewrite(bad, c.labels, w, c.supports)
    assert not r.equivalent
    assert r.inconclusive or r.residual_terms > 0
    assert not api.truth_table_equiv(bad, w)


def test_residual_is_the_word_difference():
    """Output bit k inverted: word - spec = 2^k (1 - 2 out_k), a polynomial whose
    value at every input equals the simulated word minus a*b."""
    w = 4
    c = api.gen_csa_multiplier(w)
    outs = c.aig.out_lits.copy()
    outs[0] ^= 1
    bad = api.Aig(c.aig.num_inputs, c.aig.and_lits, outs)
    r = api.backward_rewrite(bad, c.labels, w, c.supports)
    assert not r.equivalent and r.residual_terms > 0
    # evaluate the printed residual at random points against simulation
    terms = []
    for t in r.residual.split(" + "):
        f = t.split("*")
        terms.append((int(f[0]), [int(x[1:]) for x in f[1:]]))
    rng = np.random.default_rng(0)
    for _ in range(40):
        a, b = int(rng.integers(0, 1 << w)), int(rng.integers(0, 1 << w))
        inp = np.array([(a >> i) & 1 for i in range(w)] + [(b >> i) & 1 for i in range(w)], np.uint8)
        bits = api.simulate(bad, inp)
        word = sum(int(x) << k for k, x in enumerate(bits))
        val = {1 + i: int(inp[i]) for i in range(2 * w)}
        res = sum(cf * int(np.prod([val.get(v, 0) for v in vs])) if vs else cf for cf, vs in terms)
        assert res == word - a * b


def test_cap_and_argument_errors():
    c = api.gen_csa_multiplier(8)
    r = api.backward_rewrite(c.aig, np.full(c.labels.shape[0], 3, np.uint8), 8, monomial_cap=50)
    assert r.inconclusive and not r.equivalent
    with pytest.raises(ValueError, match="not a width-bit multiplier candidate"):
        api.backward_rewrite(c.aig, c.labels, 7)
    with pytest.raises(ValueError, match="labels do not cover the graph"):
        api.backward_rewrite(c.aig, c.labels[:10], 8)
    with pytest.raises(ValueError, match="width too large"):
        api.truth_table_equiv(c.aig, 11)


def test_simulate_matches_product():
    w = 7
    c = api.gen_csa_multiplier(w)
    rng = np.random.default_rng(4)
    for _ in range(50):
        a, b = int(rng.integers(0, 1 << w)), int(rng.integers(0, 1 << w))
        inp = np.array([(a >> i) & 1 for i in range(w)] + [(b >> i) & 1 for i in range(w)], np.uint8)
        bits = api.simulate(c.aig, inp)
        assert sum(int(x) << k for k, x in enumerate(bits)) == a * b


def test_csa_supports_match_generator_structure():
    s = api.csa_supports(4)
    c = api.gen_csa_multiplier(4)
    assert len(s) == 2 * 4 * 3  # one sum and one carry root per adder, w(w-1) adders
    for root, sup in s.items():
        assert c.labels[root] in (1, 2) and len(sup) in (2, 3)
        assert all((x >> 1) < root for x in sup)
