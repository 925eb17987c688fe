"""ctypes bindings to the REAL reference code (oracle/_ref/libaigsage_ref.so). TEST INFRASTRUCTURE.

The library is compiled from /root/reference's own sources by ``make -C oracle ref``
(this container only). On the GPU box only the prebuilt .so exists; ``available()``
reports whether it can be loaded.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from .pyoracle import Aig, HostGraph, Part, P, _plan_dict, dbl, i32, ptr, u32, u64

_HERE = os.path.dirname(os.path.abspath(__file__))
_PATH = os.path.join(_HERE, "_ref", "libaigsage_ref.so")
_LIB = None
REF_SRC = "/root/reference/proj/core"


def build() -> bool:
    """Compile the reference TUs + shim into oracle/_ref (needs /root/reference)."""
    if not os.path.isdir(REF_SRC):
        return os.path.exists(_PATH)
    subprocess.run(["make", "-s", "-C", _HERE, "ref"], check=True)
    return True


def available() -> bool:
    try:
        lib()
        return True
    except OSError:
        return False


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(_PATH):
            build()
        _LIB = C.CDLL(_PATH)
        _declare(_LIB)
    return _LIB


def _declare(L):
    sig = {
        "ref_last_error": (C.c_char_p, []),
        "ref_default_workers": (C.c_uint, []),
        "ref_gen_csa": (P, [u32]),
        "ref_parse_aiger": (P, [C.c_char_p]),
        "ref_aig_from_lits": (P, [u32, u32, P, u32, P]),
        "ref_aig_sizes": (None, [P, P, P, P]),
        "ref_aig_copy": (None, [P, P, P, P]),
        "ref_aig_free": (None, [P]),
        "ref_encode": (P, [P]),
        "ref_batch": (P, [P, u32]),
        "ref_graph_sizes": (None, [P, P, P, P]),
        "ref_graph_copy": (None, [P, P, P, P, P, P, P]),
        "ref_graph_free": (None, [P]),
        "ref_topo_chunks": (i32, [P, u32, P]),
        "ref_partition_multilevel": (i32, [P, u32, u64, P]),
        "ref_load_assignment": (i32, [C.c_char_p, u32, P, P]),
        "ref_regrow": (P, [P, P, u32, i32]),
        "ref_parts_sizes": (None, [P, u32, P, P, P]),
        "ref_parts_copy": (None, [P, u32, P, P, P]),
        "ref_footprint_proxy": (u64, [P]),
        "ref_materialize": (P, [P, P, u32]),
        "ref_parts_free": (None, [P]),
        "ref_crossing_fraction": (dbl, [P, P, u32]),
        "ref_build_plan": (P, [u32, P, u32, u32, u32]),
        "ref_plan_counts": (None, [P, P]),
        "ref_plan_copy": (None, [P, P, P, P, P, P]),
        "ref_plan_execute": (i32, [P, u32, P, P, P, P, u32, P, C.c_uint]),
        "ref_plan_free": (None, [P]),
        "ref_predict_full": (i32, [P, u32, u32, u32, u32, P, P, P, P, P]),
        "ref_predict_parts": (i32, [P, P, u32, u32, u32, u32, u32, u32, P, P, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args


def _err():
    return lib().ref_last_error().decode()


def _need(h):
    if not h:
        raise ValueError(_err())
    return h


class RefGraph:
    """Owns a reference ``EdaGraph`` living inside the reference library."""

    def __init__(self, handle):
        self.h = _need(handle)

    def __del__(self):
        if getattr(self, "h", None) and _LIB is not None:
            _LIB.ref_graph_free(self.h)
            self.h = None

    def sizes(self):
        n, nnz, ne = u32(), u64(), u64()
        lib().ref_graph_sizes(self.h, C.byref(n), C.byref(nnz), C.byref(ne))
        return n.value, nnz.value, ne.value

    def field(self, name: str) -> np.ndarray:
        """One EdaGraph array (row_ptr, col_idx, features, labels, degree, fwd_edges),
        copied alone so BASELINE-size graphs are compared one array at a time."""
        n, nnz, ne = self.sizes()
        shapes = {"row_ptr": (n + 1, np.uint64), "col_idx": (nnz, np.uint32), "features": ((n, 4), np.uint8),
                  "labels": (n, np.uint8), "degree": (n, np.uint32), "fwd_edges": ((ne, 2), np.uint32)}
        shape, dt = shapes[name]
        out = np.empty(shape, dt)
        args = [None] * 6
        args[list(shapes).index(name)] = out
        lib().ref_graph_copy(self.h, *[ptr(a) for a in args])
        return out

    def to_host(self) -> HostGraph:
        n, nnz, ne = self.sizes()
        rp = np.empty(n + 1, np.uint64)
        ci = np.empty(nnz, np.uint32)
        feat = np.empty((n, 4), np.uint8)
        lab = np.empty(n, np.uint8)
        deg = np.empty(n, np.uint32)
        edges = np.empty((ne, 2), np.uint32)
        lib().ref_graph_copy(self.h, ptr(rp), ptr(ci), ptr(feat), ptr(lab), ptr(deg), ptr(edges))
        return HostGraph(n, rp, ci, feat, lab, deg, edges)


def _aig_from_handle(h) -> Aig:
    ni, na, no = u32(), u32(), u32()
    lib().ref_aig_sizes(h, C.byref(ni), C.byref(na), C.byref(no))
    ands = np.empty((na.value, 2), np.uint32)
    outs = np.empty(no.value, np.uint32)
    labels = np.empty(1 + ni.value + na.value + no.value, np.uint8)
    lib().ref_aig_copy(h, ptr(ands), ptr(outs), ptr(labels))
    return Aig(ni.value, ands, outs, labels)


def gen_csa(width: int):
    """Returns (Aig, RefGraph of encode(aig))."""
    h = _need(lib().ref_gen_csa(width))
    try:
        aig = _aig_from_handle(h)
        g = RefGraph(lib().ref_encode(h))
    finally:
        lib().ref_aig_free(h)
    return aig, g


def parse_aiger(text: str):
    h = _need(lib().ref_parse_aiger(text.encode()))
    try:
        aig = _aig_from_handle(h)
        g = RefGraph(lib().ref_encode(h))
    finally:
        lib().ref_aig_free(h)
    return aig, g


def aig_from_lits(num_inputs: int, and_lits: np.ndarray, out_lits: np.ndarray):
    """Aig built through the reference's Aig::add_and/add_output; returns (Aig, RefGraph of encode)."""
    ands = np.ascontiguousarray(and_lits, np.uint32)
    outs = np.ascontiguousarray(out_lits, np.uint32)
    h = _need(lib().ref_aig_from_lits(num_inputs, ands.shape[0], ptr(ands), outs.shape[0], ptr(outs)))
    try:
        aig = _aig_from_handle(h)
        g = RefGraph(lib().ref_encode(h))
    finally:
        lib().ref_aig_free(h)
    return aig, g


def batch(g: RefGraph, copies: int) -> RefGraph:
    return RefGraph(lib().ref_batch(g.h, copies))


def topo_chunks(g: RefGraph, k: int) -> np.ndarray:
    n = g.sizes()[0]
    part = np.empty(n, np.uint32)
    if lib().ref_topo_chunks(g.h, k, ptr(part)) != 0:
        raise ValueError(_err())
    return part


def partition_multilevel(g: RefGraph, k: int, seed: int) -> np.ndarray:
    """src/partition.cpp:314-367 (does not terminate for k >= 8 on multiplier graphs)."""
    n = g.sizes()[0]
    part = np.empty(n, np.uint32)
    if lib().ref_partition_multilevel(g.h, k, seed, ptr(part)) != 0:
        raise ValueError(_err())
    return part


def load_assignment(path: str, n: int):
    part = np.empty(n, np.uint32)
    k = u32()
    st = lib().ref_load_assignment(path.encode(), n, ptr(part), C.byref(k))
    if st != 0:
        raise (ValueError if st == 1 else RuntimeError)(_err())
    return part, k.value


class RefParts:
    def __init__(self, g: RefGraph, part_of, k, with_boundary=True):
        self.g = g
        self.k = k
        part_of = np.ascontiguousarray(part_of, np.uint32)
        self.h = _need(lib().ref_regrow(g.h, ptr(part_of), k, int(with_boundary)))

    def __del__(self):
        if getattr(self, "h", None) and _LIB is not None:
            _LIB.ref_parts_free(self.h)
            self.h = None

    def part(self, p) -> Part:
        nc, nb, ne = u32(), u32(), u64()
        lib().ref_parts_sizes(self.h, p, C.byref(nc), C.byref(nb), C.byref(ne))
        core = np.empty(nc.value, np.uint32)
        bnd = np.empty(nb.value, np.uint32)
        edges = np.empty((ne.value, 2), np.uint32)
        lib().ref_parts_copy(self.h, p, ptr(core), ptr(bnd), ptr(edges))
        return Part(core, bnd, edges)

    def parts(self):
        return [self.part(p) for p in range(self.k)]

    def footprint_proxy(self) -> int:
        return int(lib().ref_footprint_proxy(self.h))

    def materialize(self, p) -> RefGraph:
        return RefGraph(lib().ref_materialize(self.g.h, self.h, p))


def crossing_fraction(g: RefGraph, part_of, k) -> float:
    return lib().ref_crossing_fraction(g.h, ptr(np.ascontiguousarray(part_of, np.uint32)), k)


def build_plan(row_ptr, hd_threshold=512, ld_threshold=12, nz_budget=96) -> dict:
    row_ptr = np.ascontiguousarray(row_ptr, np.uint64)
    rows = row_ptr.shape[0] - 1
    h = lib().ref_build_plan(rows, ptr(row_ptr), hd_threshold, ld_threshold, nz_budget)
    if not h:
        raise ValueError(_err())
    return _plan_dict(lib(), "ref", h, row_ptr, rows)


def plan_execute(plan, row_ptr, col_idx, values, dense, threads=0):
    dense = np.ascontiguousarray(dense, np.float64)
    out = np.empty((plan["rows"], dense.shape[1]), np.float64)
    st = lib().ref_plan_execute(plan["handle"], plan["rows"], ptr(row_ptr), ptr(col_idx),
                                ptr(np.ascontiguousarray(values, np.float64)), ptr(dense),
                                dense.shape[1], ptr(out), threads)
    if st != 0:
        raise ValueError(_err())
    return out


def free_plan(plan):
    lib().ref_plan_free(plan["handle"])


def predict_full(g: RefGraph, params, depth=4, in_dim=4, hidden=32, classes=5, want_logits=False):
    """Reference CPU path: make_context + run_forward (aggregation via the compiled
    spmm::execute on default_pool) + argmax. Returns (pred, confusion, accuracy, logits|None)."""
    n = g.sizes()[0]
    pred = np.empty(n, np.uint8)
    conf = np.zeros((5, 5), np.uint64)
    acc = dbl()
    lg = np.empty((n, classes), np.float64) if want_logits else None
    st = lib().ref_predict_full(g.h, depth, in_dim, hidden, classes,
                                ptr(np.ascontiguousarray(params, np.float64)), ptr(lg), ptr(pred),
                                ptr(conf), C.byref(acc))
    if st != 0:
        raise ValueError(_err())
    return pred, conf, acc.value, lg


def predict_parts(parts: RefParts, first: int, count: int, params, pred=None, depth=4, in_dim=4, hidden=32,
                  classes=5, logits=None):
    """predict (src/gnn.cpp:280-291) over parts [first, first+count), parts in parallel.
    pred (u8[n]) / logits (f64[n, classes]) receive the core rows of those parts."""
    st = lib().ref_predict_parts(parts.g.h, parts.h, first, count, depth, in_dim, hidden, classes,
                                 ptr(np.ascontiguousarray(params, np.float64)), ptr(pred), ptr(logits))
    if st != 0:
        raise ValueError(_err())


def default_workers() -> int:
    return int(lib().ref_default_workers())
