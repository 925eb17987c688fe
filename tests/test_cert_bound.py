"""The certified head's margin bound (forward.cu, GROOT_HEAD_CERT), on the CPU.

The last layer's classes-only epilogue stores x = relu(acc + b) once and lets
the tensor core take x at TF32. For any TF32 conversion of x >= 0 (truncation
or round-to-nearest), |x - tf32(x)| <= 2^-10 tf32(x), so each logit computed
from tf32(x) is within 2^-10 S_c of x.W_c, S_c = tf32(x).|W_c|. The kernel
certifies the first-maximum class when top1 - top2 > 2 * 1.125 * 2^-10 max_c S_c
(+ 1e-6 (|top1| + |top2|)); these tests check the bound holds for both
conversions and that few rows of the trained model fall back to the exact head.
"""
import os

import numpy as np

from oracle import pyoracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def tf32_trunc(x):
    return (x.astype(np.float32).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)


def tf32_rn(x):
    u = x.astype(np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x0FFF + ((u >> 13) & 1)) & 0xFFFFE000  # round to nearest even at bit 13
    return u.astype(np.uint32).view(np.float32)


def bound(S):
    return S.max(axis=1) * (2.0 * 1.125 / 1024.0)


def test_operand_bound_holds_for_truncation_and_rounding():
    rng = np.random.default_rng(3)
    x = np.abs(rng.standard_normal((20000, 32)).astype(np.float32)) * rng.uniform(0.01, 50, (20000, 1)).astype(np.float32)
    x[rng.random(x.shape) < 0.3] = 0.0  # relu zeros
    W = rng.standard_normal((32, 5)) * 0.4
    exact = x.astype(np.float64) @ W
    for conv in (tf32_trunc, tf32_rn):
        xt = conv(x).astype(np.float64)
        assert (np.abs(x - xt) <= 2.0 ** -10 * xt + 1e-45).all()
        S = xt @ np.abs(W)
        err = np.abs(xt @ W - exact)
        assert (err <= 2.0 ** -10 * S * 1.0001 + 1e-30).all()
        # a certified row keeps the exact argmax
        lg = xt @ W
        s = np.sort(lg, axis=1)
        cert = (s[:, -1] - s[:, -2]) > bound(S)
        assert cert.mean() > 0.9
        np.testing.assert_array_equal(np.argmax(lg[cert], axis=1), np.argmax(exact[cert], axis=1))


def test_trained_model_rows_needing_the_exact_head_are_rare():
    g = O.encode(O.gen_csa(64))
    prm = O.load_model(os.path.join(ROOT, "tests", "golden", "trained_csa8.asg1"))[0]
    # x = relu output of the last layer: the fp64 forward up to it, in numpy (param order:
    # per layer W_self, W_neigh, b; then W_out, b_out)
    n = g.n
    rp, ci = g.row_ptr.astype(np.int64), g.col_idx.astype(np.int64)
    deg = np.diff(rp)
    h = np.asarray(g.features, np.float64).reshape(n, 4)
    o, ind = 0, 4
    for _ in range(4):
        Ws = prm[o:o + ind * 32].reshape(ind, 32); o += ind * 32
        Wn = prm[o:o + ind * 32].reshape(ind, 32); o += ind * 32
        b = prm[o:o + 32]; o += 32
        m = np.zeros_like(h)
        np.add.at(m, np.repeat(np.arange(n), deg), h[ci])
        m /= np.maximum(deg, 1)[:, None]
        h = np.maximum(h @ Ws + m @ Wn + b, 0.0)
        ind = 32
    Wo = prm[o:o + 160].reshape(32, 5)
    bo = prm[o + 160:o + 165]
    ref = O.forward(g, prm)
    np.testing.assert_allclose(h @ Wo + bo, ref, rtol=0, atol=1e-9)
    xt = tf32_trunc(h.astype(np.float32)).astype(np.float64)
    lg = xt @ Wo + bo
    s = np.sort(lg, axis=1)
    flagged = (s[:, -1] - s[:, -2]) <= bound(xt @ np.abs(Wo)) + 1e-6 * (np.abs(s[:, -1]) + np.abs(s[:, -2]))
    assert flagged.mean() < 1e-3
    ok = ~flagged
    np.testing.assert_array_equal(np.argmax(lg[ok], axis=1), np.argmax(ref[ok], axis=1))
