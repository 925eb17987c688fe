"""The accuracy ceiling of the reference's model family on its own features
(scripts/wl_bound.py): Weisfeiler-Lehman refinement bounds every depth-L
message-passing GNN. Pins the numbers DESIGN.md §5 quotes and checks that the
reference-recipe model (tests/golden/trained_csa8.asg1, evaluated by the
oracle) stays under the bound on its training graph."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))
from wl_bound import wl_bound  # noqa: E402
from oracle import pyoracle as O  # noqa: E402


def test_wl_bound_csa():
    b8 = wl_bound(O.encode(O.gen_csa(8)), 4)
    assert [c for c, _ in b8] == [29, 75, 141, 200]
    assert abs(b8[3][1] - 0.9694) < 5e-4
    b64 = wl_bound(O.encode(O.gen_csa(64)), 4)
    assert abs(b64[3][1] - 0.8887) < 5e-4


def test_reference_model_under_bound(golden_dir):
    g = O.encode(O.gen_csa(8))
    params = O.load_model(os.path.join(golden_dir, "trained_csa8.asg1"))[0]
    pred, _, acc = O.classify(O.forward(g, params), g.labels)
    assert acc <= wl_bound(g, 4)[3][1] + 1e-12
    assert np.array_equal(pred.shape, g.labels.shape)
