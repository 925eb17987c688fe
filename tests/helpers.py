"""Shared test helpers (profiler scope names, env overrides, error/margin checks)."""
import ctypes as C
import os

import numpy as np

MARGIN_TOL = 1e-4


def profiled_names(fn):
    """Run fn with the library's per-kernel profiler on; return (result, scope names)."""
    from paper_2511_18297_b200 import _lib
    L = _lib.lib()
    L.groot_profile_enable(1)
    out = fn()
    maxk = 64
    names = C.create_string_buffer(48 * maxk)
    tot = (C.c_double * maxk)()
    cnt = (C.c_uint64 * maxk)()
    nk = C.c_uint32()
    assert L.groot_profile_read(maxk, names, tot, cnt, C.byref(nk)) == 0
    L.groot_profile_enable(0)
    got = {names.raw[48 * i:48 * (i + 1)].split(b"\0")[0].decode() for i in range(min(nk.value, maxk))}
    return out, got


def with_env(key, val, fn):
    old = os.environ.get(key)
    os.environ[key] = val
    try:
        return fn()
    finally:
        if old is None:
            del os.environ[key]
        else:
            os.environ[key] = old


def rel_err(a, ref):
    return float((np.abs(a.astype(np.float64) - ref).max(1) / np.maximum(np.abs(ref).max(1), 1e-6)).max())


def near_ties(ref_logits, tol=MARGIN_TOL):
    """Rows whose fp64 top-2 logit margin is <= tol x the row's max |logit|."""
    s = np.sort(ref_logits, axis=1)
    return (s[:, -1] - s[:, -2]) <= tol * np.maximum(np.abs(ref_logits).max(axis=1), 1e-12)


def assert_same_classes_off_ties(a, b, ref_logits, what=""):
    """Two label vectors may differ only on fp64 near-tie rows; returns the number of differences."""
    diff = a != b
    bad = diff & ~near_ties(ref_logits)
    assert not bad.any(), f"{what}: {int(bad.sum())} label differences outside fp64 near-ties"
    return int(diff.sum())
