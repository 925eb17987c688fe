"""Device training (csrc/train.cu) against the oracle restatement
of train (src/gnn.cpp:211-255, fp64) and the committed reference-recipe model.

fp64 on both sides; the device sums in fixed orders but its exp/log differ from
glibc's in the last ulp, so the bar is a tight relative tolerance (TRAIN_RTOL on
parameters after 100 Adam steps), not bit equality.
"""
import os

import numpy as np
import pytest

from oracle import pyoracle as O

pytestmark = pytest.mark.gpu

TRAIN_RTOL = 1e-7


@pytest.fixture(scope="module")
def api():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2511_18297_b200 import api as A
    return A


def graph(api, width, copies=1):
    c = api.gen_csa_multiplier(width)
    g = api.encode(c.aig, c.labels)
    return api.batch(g, copies) if copies > 1 else g


def test_reference_recipe_reproduces_committed_model(api, golden_dir):
    """8-bit CSA, 100 epochs, lr 1e-3, Adam, seed 7 (inc/gnn.hpp:38-45) == trained_csa8.asg1."""
    import json
    g = graph(api, 8)
    st = api.TrainStats(None, None)
    model = api.train(g, epochs=100, learning_rate=1e-3, seed=7, stats=st)
    ref = O.load_model(os.path.join(golden_dir, "trained_csa8.asg1"))[0]
    np.testing.assert_allclose(model.params, ref, rtol=TRAIN_RTOL, atol=1e-12)
    meta = json.load(open(os.path.join(golden_dir, "trained_csa8.json")))
    assert abs(st.loss[-1] - meta["final_loss"]) <= 1e-9 * abs(meta["final_loss"])
    assert st.accuracy[-1] == pytest.approx(meta["final_train_accuracy"], abs=1e-12)
    assert np.all(np.diff(st.loss[:20]) < 0)  # the loss falls over the first epochs


@pytest.mark.parametrize("width,copies,epochs,lr", [(4, 1, 5, 1e-2), (16, 2, 20, 3e-3)])
def test_train_matches_oracle(api, width, copies, epochs, lr):
    g = graph(api, width, copies)
    h = O.batch(O.encode(O.gen_csa(width)), copies) if copies > 1 else O.encode(O.gen_csa(width))
    prm, loss, acc = O.train(h, epochs=epochs, lr=lr, seed=3)
    st = api.TrainStats(None, None)
    model = api.train(g, epochs=epochs, learning_rate=lr, seed=3, stats=st)
    np.testing.assert_allclose(model.params, prm, rtol=TRAIN_RTOL, atol=1e-12)
    assert abs(st.loss[-1] - loss) <= 1e-9 * abs(loss)
    assert st.accuracy[-1] == pytest.approx(acc, abs=1e-12)


def test_loss_and_grads_and_grad_check(api):
    """Analytic gradient vs central differences (SPEC acceptance #11, inc/gnn.hpp:88-90),
    on a depth-2, hidden-8 model of a 4-bit CSA (every parameter checked)."""
    g = graph(api, 4)
    # perturbed so no pre-activation sits exactly on the ReLU kink (zero biases put
    # the isolated constant node's z at 0, where central differences are one-sided)
    prm = O.init_model(5, hidden=8, depth=2) + np.random.default_rng(1).normal(0, 0.05, O.param_count(2, 4, 8, 5))
    loss, grads = api.loss_and_grads(prm, g, depth=2, hidden=8)
    assert np.isfinite(loss) and grads.shape == prm.shape and np.abs(grads).max() > 0
    assert api.grad_check(prm, g, epsilon=1e-5, depth=2, hidden=8) <= 1e-6


def test_train_errors(api):
    g = graph(api, 4)
    with pytest.raises(ValueError, match="learning rate must be positive"):
        api.train(g, epochs=1, learning_rate=0.0)


def test_verify_from_predicted_classes(api, golden_dir):
    """The paper's loop: classes predicted on the device by the
    device-trained model drive backward_rewrite to prove 8/16/32-bit CSA
    multipliers; the same classes on a mutated multiplier give a nonzero residual."""
    model = api.load_model(os.path.join(golden_dir, "trained_csa64_gpu.asg1"))
    for w in (8, 16, 32):
        c = api.gen_csa_multiplier(w)
        pred = api.predict_full(model, api.encode(c.aig, c.labels))
        rep = api.backward_rewrite(c.aig, pred.labels, w)
        assert rep.equivalent and not rep.inconclusive, (w, rep)
        assert rep.shortcut_count > 0
    c = api.gen_csa_multiplier(8)
    pred = api.predict_full(model, api.encode(c.aig, c.labels))
    bad = api.Aig(c.aig.num_inputs, c.aig.and_lits.copy(), c.aig.out_lits.copy())
    bad.and_lits[len(bad.and_lits) // 2, 0] ^= 1  # one inverted fan-in
    rep = api.backward_rewrite(bad, pred.labels, 8)
    assert not rep.equivalent and rep.residual_terms > 0
    assert not api.truth_table_equiv(bad, 8)
