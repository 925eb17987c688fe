"""Radix-4 Booth multiplier generator (BASELINE config 3).

The reference has no Booth generator, so the generator is
pinned by what a multiplier must do and by the reference's own code downstream:
* functional: bit-parallel simulation of the AIG multiplies (exhaustive for
  small widths, random operands up to 64 bits);
* well-formed: the reference's own Aig::add_and / add_output accept it (fanins
  strictly below the node), its encode equals the oracle's, and our AIGER text
  round-trips through our parser;
* deterministic: sha256 of the generated arrays pinned in tests/golden/booth_digests.json.
Device-side parity (encode / batch / regrow / forward on Booth graphs) is in
tests/test_gpu_parity.py.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import pyoracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def api():
    from paper_2511_18297_b200 import _lib, api as A
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2511_18297_b200 import build
        build.build()
    return A


def simulate(aig, a_vals, b_vals, w):
    """Bit-parallel AIG simulation: operands as Python ints, 64 patterns per word."""
    npat = len(a_vals)
    words = (npat + 63) // 64
    ni = aig.num_inputs
    na = aig.num_ands
    vals = np.zeros((1 + ni + na, words), np.uint64)
    for bit in range(w):
        for s in range(npat):
            wi, bi = divmod(s, 64)
            if (a_vals[s] >> bit) & 1:
                vals[1 + bit, wi] |= np.uint64(1) << np.uint64(bi)
            if (b_vals[s] >> bit) & 1:
                vals[1 + w + bit, wi] |= np.uint64(1) << np.uint64(bi)
    full = np.uint64(0xFFFFFFFFFFFFFFFF)
    lits = aig.and_lits.astype(np.int64)
    for k in range(na):
        lv, rv = vals[lits[k, 0] >> 1], vals[lits[k, 1] >> 1]
        if lits[k, 0] & 1:
            lv = lv ^ full
        if lits[k, 1] & 1:
            rv = rv ^ full
        vals[1 + ni + k] = lv & rv
    prods = []
    for s in range(npat):
        wi, bi = divmod(s, 64)
        p = 0
        for k, o in enumerate(aig.out_lits.astype(np.int64)):
            bit = (int(vals[o >> 1, wi]) >> bi) & 1
            p |= (bit ^ int(o & 1)) << k
        prods.append(p)
    return prods


@pytest.mark.parametrize("w", [2, 3, 4, 5])
def test_booth_exhaustive(api, w):
    c = api.gen_booth_multiplier(w)
    pairs = [(x, y) for x in range(1 << w) for y in range(1 << w)]
    got = simulate(c.aig, [p[0] for p in pairs], [p[1] for p in pairs], w)
    assert got == [x * y for x, y in pairs]


@pytest.mark.parametrize("w", [8, 13, 16, 33, 64])
def test_booth_random_operands(api, w):
    c = api.gen_booth_multiplier(w)
    rng = np.random.default_rng(w)
    a = [int(x) for x in rng.integers(0, 1 << min(w, 62), 128)]
    b = [int(x) for x in rng.integers(0, 1 << min(w, 62), 128)]
    if w == 64:  # cover the top bits too
        a[:4] = [(1 << 64) - 1, 1 << 63, (1 << 64) - 1, 12345]
        b[:4] = [(1 << 64) - 1, (1 << 64) - 1, 1, 1 << 63]
    assert simulate(c.aig, a, b, w) == [x * y for x, y in zip(a, b)]


@pytest.mark.parametrize("w", [4, 16, 64])
def test_booth_structure_and_labels(api, w):
    c = api.gen_booth_multiplier(w)
    n_nodes = c.aig.num_nodes
    assert c.aig.num_inputs == 2 * w and c.aig.out_lits.shape[0] == 2 * w
    lits = c.aig.and_lits
    own = np.arange(1 + 2 * w, n_nodes, dtype=np.int64)
    assert ((lits[:, 0] >> 1) < own).all() and ((lits[:, 1] >> 1) < own).all(), "fanins strictly lower"
    assert ((lits >> 1) > 0).all(), "no constant fanins (constants are folded)"
    lab = c.labels
    assert lab.shape[0] == n_nodes + 2 * w
    assert lab[0] == 3 and (lab[1:1 + 2 * w] == 4).all() and (lab[n_nodes:] == 0).all()
    hist = np.bincount(lab[1 + 2 * w:n_nodes], minlength=5)
    assert hist[1] > 0 and hist[2] > 0 and hist[3] > 0 and hist[0] == 0 and hist[4] == 0


def test_booth_reference_aig_and_encode(api):
    """The reference's own Aig::add_and validation and encode (compiled from
    /root/reference) accept the Booth AIG; encode equals the oracle's, and our
    AIGER text round-trips through our parser."""
    from oracle import pyref
    if not pyref.available():
        pytest.skip("reference build (oracle/_ref) not available")
    c = api.gen_booth_multiplier(16)
    back = api.parse_aiger(api.write_aiger(c.aig))
    np.testing.assert_array_equal(back.and_lits, c.aig.and_lits)
    np.testing.assert_array_equal(back.out_lits, c.aig.out_lits)
    raig, rg = pyref.aig_from_lits(c.aig.num_inputs, c.aig.and_lits, c.aig.out_lits)
    np.testing.assert_array_equal(raig.and_lits, c.aig.and_lits)
    np.testing.assert_array_equal(raig.out_lits, c.aig.out_lits)
    og = O.encode(O.Aig(c.aig.num_inputs, c.aig.and_lits, c.aig.out_lits, c.labels))
    rh = rg.to_host()
    for f in ("row_ptr", "col_idx", "features", "degree", "fwd_edges"):
        np.testing.assert_array_equal(getattr(rh, f), getattr(og, f), err_msg=f)


def test_booth_digests(api, golden_dir):
    with open(os.path.join(golden_dir, "booth_digests.json")) as f:
        dig = json.load(f)
    assert dig, "booth digests missing"
    for w, want in dig.items():
        c = api.gen_booth_multiplier(int(w))
        h = hashlib.sha256()
        for arr in (c.aig.and_lits, c.aig.out_lits, c.labels):
            h.update(np.ascontiguousarray(arr).tobytes())
        assert h.hexdigest() == want, f"booth {w}"
