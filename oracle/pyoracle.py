"""ctypes bindings to the oracle restatement (oracle/liboracle.so). TEST INFRASTRUCTURE.

Every wrapper names the reference function it restates; see oracle.h for the
file:line citations. Arrays are numpy; graphs are ``HostGraph`` records.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def build() -> str:
    """Compile liboracle.so (g++ only; no /root/reference needed)."""
    subprocess.run(["make", "-s", "-C", _HERE, "liboracle.so"], check=True)
    return os.path.join(_HERE, "liboracle.so")


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        src = os.path.join(_HERE, "oracle.cpp")
        if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
            build()
        _LIB = C.CDLL(path)
        _declare(_LIB)
    return _LIB


P = C.c_void_p
u32, u64, dbl, i32 = C.c_uint32, C.c_uint64, C.c_double, C.c_int


def _declare(L):
    sig = {
        "orc_csa_sizes": (i32, [u32, P, P, P]),
        "orc_gen_csa": (i32, [u32, P, P, P]),
        "orc_encode": (i32, [u32, u32, P, u32, P, P, P, P, P, P]),
        "orc_build_csr": (i32, [u32, u64, P, P, P]),
        "orc_batch": (i32, [u32, u64, P, P, P, P, P, u32, P, P, P, P, P, P]),
        "orc_topo_chunks": (i32, [u32, u32, P]),
        "orc_regrow": (P, [u32, P, P, u64, P, P, u32, i32]),
        "orc_parts_count": (u32, [P]),
        "orc_parts_sizes": (None, [P, u32, P, P, P]),
        "orc_parts_copy": (None, [P, u32, P, P, P]),
        "orc_parts_free": (None, [P]),
        "orc_crossing_fraction": (dbl, [u64, P, P]),
        "orc_edge_cut": (u64, [u64, P, P]),
        "orc_degree_sort": (i32, [u32, P, P, P]),
        "orc_build_plan": (P, [u32, P, u32, u32, u32]),
        "orc_plan_counts": (None, [P, P]),
        "orc_plan_copy": (None, [P, P, P, P, P, P]),
        "orc_plan_execute": (i32, [P, u32, P, P, P, P, u32, P]),
        "orc_plan_free": (None, [P]),
        "orc_reference_spmm": (i32, [u32, P, P, P, P, u32, P]),
        "orc_param_count": (u64, [u32, u32, u32, u32]),
        "orc_init_model": (i32, [u64, u32, u32, u32, u32, P]),
        "orc_forward": (i32, [u32, P, P, P, u32, u32, u32, u32, P, P, C.c_uint]),
        "orc_classify": (i32, [u32, u32, P, P, P, P, P]),
        "orc_train": (i32, [u32, P, P, P, P, u32, dbl, u64, P, P, P]),
        "orc_last_error": (C.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args


def ptr(a):
    return None if a is None else a.ctypes.data_as(P)


class OracleError(RuntimeError):
    pass


def _check(st):
    if st != 0:
        msg = lib().orc_last_error().decode()
        raise (ValueError if st == 1 else OracleError)(msg)


@dataclass
class Aig:
    """Flat AIG: and_lits (A,2) u32 literals 2v+inv; out_lits (O,) u32; labels (n,) u8."""
    num_inputs: int
    and_lits: np.ndarray
    out_lits: np.ndarray
    labels: np.ndarray

    @property
    def num_ands(self):
        return int(self.and_lits.shape[0])

    @property
    def num_outputs(self):
        return int(self.out_lits.shape[0])

    @property
    def num_nodes(self):
        return 1 + self.num_inputs + self.num_ands


@dataclass
class HostGraph:
    """EdaGraph (inc/encode.hpp:18-31) as numpy arrays."""
    n: int
    row_ptr: np.ndarray      # u64 [n+1]
    col_idx: np.ndarray      # u32 [nnz]
    features: np.ndarray     # u8 [n,4]
    labels: np.ndarray       # u8 [n]
    degree: np.ndarray       # u32 [n]
    fwd_edges: np.ndarray    # u32 [E,2]

    @property
    def nnz(self):
        return int(self.row_ptr[-1])

    @property
    def num_edges(self):
        return int(self.fwd_edges.shape[0])


@dataclass
class Part:
    """AugmentedPartition (inc/partition.hpp:23-33)."""
    core_nodes: np.ndarray
    boundary_nodes: np.ndarray
    edges: np.ndarray  # u32 [E,2] local ids

    @property
    def local_to_global(self):
        return np.concatenate([self.core_nodes, self.boundary_nodes])

    @property
    def num_core(self):
        return int(self.core_nodes.shape[0])

    @property
    def core_mask(self):
        m = np.zeros(self.local_to_global.shape[0], np.uint8)
        m[: self.num_core] = 1
        return m


def gen_csa(width: int) -> Aig:
    """gen_csa_multiplier (src/circuitgen.cpp:66-133)."""
    ni, na, no = u32(), u32(), u32()
    _check(lib().orc_csa_sizes(width, C.byref(ni), C.byref(na), C.byref(no)))
    ands = np.empty((na.value, 2), np.uint32)
    outs = np.empty(no.value, np.uint32)
    labels = np.empty(1 + ni.value + na.value + no.value, np.uint8)
    _check(lib().orc_gen_csa(width, ptr(ands), ptr(outs), ptr(labels)))
    return Aig(ni.value, ands, outs, labels)


def encode(aig: Aig) -> HostGraph:
    """encode (src/encode.cpp:33-68)."""
    n = aig.num_nodes + aig.num_outputs
    if aig.labels.shape[0] != n:
        raise ValueError("encode: label count does not match encoded node count")
    E = 2 * aig.num_ands + aig.num_outputs
    feat = np.empty((n, 4), np.uint8)
    edges = np.empty((E, 2), np.uint32)
    rp = np.empty(n + 1, np.uint64)
    ci = np.empty(2 * E, np.uint32)
    deg = np.empty(n, np.uint32)
    ands = np.ascontiguousarray(aig.and_lits, np.uint32)
    outs = np.ascontiguousarray(aig.out_lits, np.uint32)
    _check(lib().orc_encode(aig.num_inputs, aig.num_ands, ptr(ands), aig.num_outputs, ptr(outs),
                            ptr(feat), ptr(edges), ptr(rp), ptr(ci), ptr(deg)))
    return HostGraph(n, rp, ci, feat, aig.labels.copy(), deg, edges)


def build_csr(n: int, edges: np.ndarray):
    """build_symmetric_csr (src/encode.cpp:14-31)."""
    edges = np.ascontiguousarray(edges, np.uint32)
    rp = np.empty(n + 1, np.uint64)
    ci = np.empty(2 * edges.shape[0], np.uint32)
    _check(lib().orc_build_csr(n, edges.shape[0], ptr(edges), ptr(rp), ptr(ci)))
    return rp, ci


def batch(g: HostGraph, copies: int) -> HostGraph:
    """batch (src/encode.cpp:70-101)."""
    if copies < 1:
        raise ValueError("batch: copy count must be >= 1")
    if copies == 1:
        return g
    n = g.n * copies
    rp = np.empty(n + 1, np.uint64)
    ci = np.empty(g.nnz * copies, np.uint32)
    feat = np.empty((n, 4), np.uint8)
    lab = np.empty(n, np.uint8)
    deg = np.empty(n, np.uint32)
    edges = np.empty((g.num_edges * copies, 2), np.uint32)
    _check(lib().orc_batch(g.n, g.num_edges, ptr(g.row_ptr), ptr(g.col_idx), ptr(g.features),
                           ptr(g.labels), ptr(g.fwd_edges), copies, ptr(rp), ptr(ci), ptr(feat),
                           ptr(lab), ptr(deg), ptr(edges)))
    return HostGraph(n, rp, ci, feat, lab, deg, edges)


def topo_chunks(n: int, k: int) -> np.ndarray:
    """partition_topo_chunks (src/partition.cpp:301-312)."""
    part = np.empty(n, np.uint32)
    _check(lib().orc_topo_chunks(n, k, ptr(part)))
    return part


def regrow(g: HostGraph, part_of: np.ndarray, k: int, with_boundary: bool = True):
    """regrow / core_subgraphs (src/partition.cpp:402-466)."""
    part_of = np.ascontiguousarray(part_of, np.uint32)
    h = lib().orc_regrow(g.n, ptr(g.row_ptr), ptr(g.col_idx), g.num_edges, ptr(g.fwd_edges),
                         ptr(part_of), k, int(with_boundary))
    if not h:
        raise ValueError(lib().orc_last_error().decode())
    out = []
    try:
        for p in range(lib().orc_parts_count(h)):
            nc, nb, ne = u32(), u32(), u64()
            lib().orc_parts_sizes(h, p, C.byref(nc), C.byref(nb), C.byref(ne))
            core = np.empty(nc.value, np.uint32)
            bnd = np.empty(nb.value, np.uint32)
            edges = np.empty((ne.value, 2), np.uint32)
            lib().orc_parts_copy(h, p, ptr(core), ptr(bnd), ptr(edges))
            out.append(Part(core, bnd, edges))
    finally:
        lib().orc_parts_free(h)
    return out


def materialize(g: HostGraph, part: Part) -> HostGraph:
    """materialize (src/partition.cpp:488-506)."""
    l2g = part.local_to_global
    n = int(l2g.shape[0])
    rp, ci = build_csr(n, part.edges)
    deg = np.diff(rp).astype(np.uint32)
    return HostGraph(n, rp, ci, g.features[l2g].copy(), g.labels[l2g].copy(), deg, part.edges.copy())


def crossing_fraction(g: HostGraph, part_of: np.ndarray) -> float:
    """crossing_fraction (src/partition.cpp:468-474)."""
    part_of = np.ascontiguousarray(part_of, np.uint32)
    return lib().orc_crossing_fraction(g.num_edges, ptr(g.fwd_edges), ptr(part_of))


def edge_cut(g: HostGraph, part_of: np.ndarray) -> int:
    """edge_cut (src/partition.cpp:508-513)."""
    part_of = np.ascontiguousarray(part_of, np.uint32)
    return lib().orc_edge_cut(g.num_edges, ptr(g.fwd_edges), ptr(part_of))


def footprint_proxy(parts, feature_cols: int = 4, hidden_dim: int = 32) -> int:
    """footprint_proxy (src/partition.cpp:476-486)."""
    best = 0
    for p in parts:
        size = int(p.core_nodes.shape[0] + p.boundary_nodes.shape[0])
        best = max(best, size * (feature_cols + hidden_dim) * 4 + 2 * int(p.edges.shape[0]) * 8)
    return best


def degree_sort(row_ptr: np.ndarray):
    """degree_sort (src/spmm.cpp:9-35)."""
    rows = row_ptr.shape[0] - 1
    perm = np.empty(rows, np.uint32)
    srp = np.empty(rows + 1, np.uint64)
    _check(lib().orc_degree_sort(rows, ptr(row_ptr), ptr(perm), ptr(srp)))
    return perm, srp


def build_plan(row_ptr: np.ndarray, hd_threshold=512, ld_threshold=12, nz_budget=96) -> dict:
    """build_plan (src/spmm.cpp:37-127) -> dict of numpy arrays."""
    rows = row_ptr.shape[0] - 1
    row_ptr = np.ascontiguousarray(row_ptr, np.uint64)
    h = lib().orc_build_plan(rows, ptr(row_ptr), hd_threshold, ld_threshold, nz_budget)
    if not h:
        raise ValueError(lib().orc_last_error().decode())
    return _plan_dict(lib(), "orc", h, row_ptr, rows)


def _plan_dict(L, pre, h, row_ptr, rows):
    c = np.zeros(6, np.uint64)
    getattr(L, pre + "_plan_counts")(h, ptr(c))
    hd = np.empty(int(c[0]), np.uint32)
    mid = np.empty(int(c[1]), np.uint32)
    ldg = np.empty((int(c[2]), 3), np.uint32)
    units = np.empty((int(c[3]), 6), np.uint64)
    perm = np.empty(rows, np.uint32)
    getattr(L, pre + "_plan_copy")(h, ptr(hd), ptr(mid), ptr(ldg), ptr(units), ptr(perm))
    return {"handle": h, "rows": rows, "hd_rows": hd, "mid_rows": mid, "ld_groups": ldg,
            "units": units, "perm": perm, "ld_row_begin": int(c[4]), "ld_row_end": int(c[5])}


def plan_execute(plan: dict, row_ptr, col_idx, values, dense: np.ndarray) -> np.ndarray:
    """spmm::execute (inc/spmm.hpp:106-181), fp64."""
    dense = np.ascontiguousarray(dense, np.float64)
    f = dense.shape[1]
    out = np.empty((plan["rows"], f), np.float64)
    _check(lib().orc_plan_execute(plan["handle"], plan["rows"], ptr(row_ptr), ptr(col_idx),
                                  ptr(np.ascontiguousarray(values, np.float64)), ptr(dense), f,
                                  ptr(out)))
    return out


def free_plan(plan: dict):
    lib().orc_plan_free(plan["handle"])


def reference_spmm(row_ptr, col_idx, values, dense):
    """reference_spmm (inc/spmm.hpp:184-195)."""
    dense = np.ascontiguousarray(dense, np.float64)
    rows = row_ptr.shape[0] - 1
    out = np.empty((rows, dense.shape[1]), np.float64)
    _check(lib().orc_reference_spmm(rows, ptr(row_ptr), ptr(col_idx),
                                    ptr(np.ascontiguousarray(values, np.float64)), ptr(dense),
                                    dense.shape[1], ptr(out)))
    return out


def param_count(depth=4, in_dim=4, hidden=32, classes=5) -> int:
    return int(lib().orc_param_count(depth, in_dim, hidden, classes))


def init_model(seed: int, in_dim=4, hidden=32, classes=5, depth=4) -> np.ndarray:
    """init_model (src/gnn.cpp:113-138): flat params in ASG1 order."""
    prm = np.empty(param_count(depth, in_dim, hidden, classes), np.float64)
    _check(lib().orc_init_model(seed, in_dim, hidden, classes, depth, ptr(prm)))
    return prm


def forward(g: HostGraph, params: np.ndarray, depth=4, in_dim=4, hidden=32, classes=5,
            threads: int = 0) -> np.ndarray:
    """forward (src/gnn.cpp:172-178) fp64 logits [n, classes]."""
    logits = np.empty((g.n, classes), np.float64)
    _check(lib().orc_forward(g.n, ptr(g.row_ptr), ptr(g.col_idx),
                             ptr(np.ascontiguousarray(g.features, np.uint8)), depth, in_dim,
                             hidden, classes, ptr(np.ascontiguousarray(params, np.float64)),
                             ptr(logits), threads))
    return logits


def classify(logits: np.ndarray, truth: np.ndarray | None = None):
    """score_rows + finish_prediction (src/gnn.cpp:259-276): (pred, confusion, accuracy)."""
    logits = np.ascontiguousarray(logits, np.float64)
    n, k = logits.shape
    pred = np.empty(n, np.uint8)
    conf = np.zeros((5, 5), np.uint64)
    acc = dbl()
    _check(lib().orc_classify(n, k, ptr(logits), ptr(truth), ptr(pred), ptr(conf), C.byref(acc)))
    return pred, conf, acc.value


def predict_full(g: HostGraph, params, depth=4):
    """predict_full (src/gnn.cpp:293-300)."""
    lg = forward(g, params, depth=depth)
    pred, conf, acc = classify(lg, g.labels)
    return pred, conf, acc, lg


def predict(g: HostGraph, parts, params, depth=4):
    """predict (src/gnn.cpp:280-291): each node scored from its core partition."""
    pred = np.zeros(g.n, np.uint8)
    for p in parts:
        sub = materialize(g, p)
        lg = forward(sub, params, depth=depth)
        pp, _, _ = classify(lg)
        pred[p.core_nodes] = pp[: p.num_core]
    conf = np.zeros((5, 5), np.uint64)
    np.add.at(conf, (g.labels.astype(np.int64), pred.astype(np.int64)), 1)
    acc = float((pred == g.labels).sum()) / g.n if g.n else 0.0
    return pred, conf, acc


def train(g: HostGraph, epochs=100, lr=1e-3, seed=7):
    """train (src/gnn.cpp:211-255): returns (params, final_loss, final_train_accuracy)."""
    prm = np.empty(param_count(), np.float64)
    fl, fa = dbl(), dbl()
    _check(lib().orc_train(g.n, ptr(g.row_ptr), ptr(g.col_idx), ptr(g.features), ptr(g.labels),
                           epochs, lr, seed, ptr(prm), C.byref(fl), C.byref(fa)))
    return prm, fl.value, fa.value


# --- ASG1 model files (src/gnn.cpp:330-372) ---------------------------------
def save_model(path: str, params: np.ndarray, depth=4, in_dim=4, hidden=32, classes=5):
    with open(path, "wb") as f:
        f.write(b"ASG1")
        f.write(np.array([depth, in_dim, hidden, classes], np.uint32).tobytes())
        f.write(np.ascontiguousarray(params, np.float64).tobytes())


def load_model(path: str):
    with open(path, "rb") as f:
        data = f.read()
    if data[:4] != b"ASG1":
        raise OracleError("model file: bad magic or version")
    depth, in_dim, hidden, classes = (int(x) for x in np.frombuffer(data[4:20], np.uint32))
    cnt = param_count(depth, in_dim, hidden, classes)
    prm = np.frombuffer(data[20:20 + 8 * cnt], np.float64).copy()
    if prm.shape[0] != cnt:
        raise OracleError("model file: truncated")
    return prm, dict(depth=depth, in_dim=in_dim, hidden=hidden, classes=classes)


# ---------------------------------------------------------------------------
# partition_multilevel replacement. The reference's
# partition_multilevel (src/partition.cpp:314-367) livelocks in rebalance
# (:259-297) for k >= 8 on multiplier graphs; its result is the cheaper of a
# multilevel cut and the topo chunks refined by greedy boundary moves
# (:357-366). This restates the device algorithm that replaces it (numpy,
# test infrastructure): start from the topo chunks, then rounds of
# deterministic size-constrained label propagation --
#   * every node v picks the neighbouring part t != part(v) with the most
#     neighbours (ties: lowest id), allowed only upward (t > part(v)) in even
#     rounds and downward in odd rounds; gain = conn(t) - conn(part(v)) > 0;
#   * candidates moving into t are ranked by (gain desc, node id asc) and the
#     first cap - weight(t) of them move (cap = ceil(1.05 n / k),
#     src/partition.cpp:328-329), weights taken at the round's start;
#   * a part that would lose all its nodes keeps every node that round;
#   * stop after two consecutive rounds without a move, or max_rounds.
# Every round keeps every part within the cap and nonempty, so it terminates
# for any k. On graphs where the reference terminates (k <= 4 on CSA) the
# result equals partition_multilevel's bit for bit (tests/test_oracle.py).
# ---------------------------------------------------------------------------
def lp_cap(n: int, k: int) -> int:
    """ceil(1.05 * n / k) in double, as src/partition.cpp:328-329."""
    return int(np.ceil(1.05 * float(n) / k))


def partition_lp(row_ptr, col_idx, n: int, k: int, max_rounds: int = 32) -> np.ndarray:
    if k < 1:
        raise ValueError("partition: k must be >= 1")
    if k > n:
        raise ValueError("partition: k exceeds node count")
    part = topo_chunks(n, k).astype(np.int64)
    if k == 1:
        return part.astype(np.uint32)
    cap = lp_cap(n, k)
    rp = np.asarray(row_ptr, np.int64)
    ci = np.asarray(col_idx, np.int64)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
    idle = 0
    for it in range(max_rounds):
        key = rows * k + part[ci]
        uk, cnt = np.unique(key, return_counts=True)
        v, p = uk // k, uk % k
        own = np.zeros(n, np.int64)
        m = p == part[v]
        own[v[m]] = cnt[m]
        d = (p > part[v]) if it % 2 == 0 else (p < part[v])
        vv, pp, cc = v[d], p[d], cnt[d]
        o = np.lexsort((pp, -cc, vv))           # per node: most neighbours, then lowest part
        vv, pp, cc = vv[o], pp[o], cc[o]
        first = np.ones(vv.size, bool)
        first[1:] = vv[1:] != vv[:-1]
        vv, pp, gain = vv[first], pp[first], cc[first] - own[vv[first]]
        g = gain > 0
        vv, pp, gain = vv[g], pp[g], gain[g]
        w = np.bincount(part, minlength=k)
        room = np.maximum(cap - w, 0)
        o = np.lexsort((vv, -gain, pp))         # per target part: gain desc, node asc
        vv, pp, gain = vv[o], pp[o], gain[o]
        rank = np.arange(vv.size) - np.searchsorted(pp, pp)
        ok = rank < room[pp]
        vv, pp = vv[ok], pp[ok]
        out = np.bincount(part[vv], minlength=k)
        keep = out >= w                          # a part would be emptied: none of its nodes move
        mv = ~keep[part[vv]]
        vv, pp = vv[mv], pp[mv]
        part[vv] = pp
        idle = 0 if vv.size else idle + 1
        if idle >= 2:
            break
    return part.astype(np.uint32)
