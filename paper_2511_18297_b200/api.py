"""Python mirror of the reference operator API (namespace aigsage) over the C ABI.

Same function names, argument meaning and error behaviour as
/root/reference/proj/core/include/aigsage/*.hpp for the hot path:
AIG load -> feature build -> partition -> edge re-growth -> layer forward ->
classify. Graphs, assignments, partitions and models live in HBM behind opaque
handles; numpy arrays appear only at the edges (inputs / copy-outs).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import GrootError, GrootInvalidArgument, check, lib, ptr  # noqa: F401

NUM_CLASSES = 5


NODE_CLASS = {"PO": 0, "MAJ": 1, "XOR": 2, "AND": 3, "PI": 4}  # inc/circuitgen.hpp:15


# ---------------------------------------------------------------------------
# AIG (inc/aig.hpp) and sources (src/circuitgen.cpp, src/aig.cpp)
# ---------------------------------------------------------------------------
@dataclass
class Aig:
    """And-Inverter Graph: node 0 const, inputs 1..I, ANDs after (inc/aig.hpp:30-33).
    and_lits: (A,2) u32 literals 2v+inv; out_lits: (O,) u32."""
    num_inputs: int
    and_lits: np.ndarray
    out_lits: np.ndarray

    @property
    def num_ands(self) -> int:
        return int(self.and_lits.shape[0])

    @property
    def num_nodes(self) -> int:
        return 1 + self.num_inputs + self.num_ands

    @property
    def first_and(self) -> int:
        return 1 + self.num_inputs


@dataclass
class CsaCircuit:
    """gen_csa_multiplier result (inc/circuitgen.hpp:27-33): aig + GroundTruth labels.
    `supports` (GroundTruth::supports: adder root -> support literals) is built on
    first access for CSA circuits."""
    aig: Aig
    labels: np.ndarray
    width: int
    kind: str = "csa"
    _supports: dict | None = field(default=None, repr=False)

    @property
    def supports(self) -> dict:
        if self._supports is None:
            self._supports = csa_supports(self.width) if self.kind == "csa" else {}
        return self._supports


def csa_supports(width: int) -> dict:
    """GroundTruth::supports of gen_csa_multiplier (src/circuitgen.cpp:30-32, 50-62):
    {root node: [support literals 2v+inv]}."""
    cnt = C.c_uint32()
    check(lib().groot_csa_supports(width, C.byref(cnt), None))
    rec = np.empty((cnt.value, 5), np.uint32)
    check(lib().groot_csa_supports(width, C.byref(cnt), ptr(rec)))
    return {int(r[0]): [int(x) for x in r[2:2 + int(r[1])]] for r in rec}


def gen_csa_multiplier(width: int) -> CsaCircuit:
    """src/circuitgen.cpp:66-133."""
    ni, na, no = C.c_uint32(), C.c_uint32(), C.c_uint32()
    check(lib().groot_csa_sizes(width, C.byref(ni), C.byref(na), C.byref(no)))
    ands = np.empty((na.value, 2), np.uint32)
    outs = np.empty(no.value, np.uint32)
    labels = np.empty(1 + ni.value + na.value + no.value, np.uint8)
    check(lib().groot_gen_csa(width, ptr(ands), ptr(outs), ptr(labels)))
    return CsaCircuit(Aig(ni.value, ands, outs), labels, width)


def gen_booth_multiplier(width: int) -> CsaCircuit:
    """Radix-4 Booth multiplier AIG (BASELINE config 3; the reference has no
    Booth generator). Same conventions as gen_csa_multiplier:
    PIs a = 1..w, b = w+1..2w, POs = the 2w product bits, labels PO/MAJ/XOR/AND/PI."""
    ni, na, no = C.c_uint32(), C.c_uint32(), C.c_uint32()
    check(lib().groot_booth_sizes(width, C.byref(ni), C.byref(na), C.byref(no)))
    ands = np.empty((na.value, 2), np.uint32)
    outs = np.empty(no.value, np.uint32)
    labels = np.empty(1 + ni.value + na.value + no.value, np.uint8)
    check(lib().groot_gen_booth(width, ptr(ands), ptr(outs), ptr(labels)))
    return CsaCircuit(Aig(ni.value, ands, outs), labels, width, "booth")


def parse_aiger(text: str | bytes) -> Aig:
    """src/aig.cpp:47-88 (ASCII 'aag', latches rejected, same error texts)."""
    data = text.encode() if isinstance(text, str) else bytes(text)
    ni, na, no = C.c_uint32(), C.c_uint32(), C.c_uint32()
    check(lib().groot_aiger_sizes(data, len(data), C.byref(ni), C.byref(na), C.byref(no)))
    ands = np.empty((na.value, 2), np.uint32)
    outs = np.empty(no.value, np.uint32)
    check(lib().groot_aiger_fill(data, len(data), ptr(ands), ptr(outs)))
    return Aig(ni.value, ands, outs)


def parse_aiger_file(path: str) -> Aig:
    try:
        with open(path, "rb") as f:
            return parse_aiger(f.read())
    except OSError as e:
        raise GrootError(2, f"cannot open AIGER file: {path}") from e


def write_aiger(aig: Aig) -> str:
    """src/aig.cpp:96-113."""
    i, a = aig.num_inputs, aig.num_ands
    lines = [f"aag {i + a} {i} 0 {aig.out_lits.shape[0]} {a}"]
    lines += [str(2 * (k + 1)) for k in range(i)]
    lines += [str(int(x)) for x in aig.out_lits]
    lines += [f"{2 * (i + 1 + k)} {int(l)} {int(r)}" for k, (l, r) in enumerate(aig.and_lits)]
    return "\n".join(lines) + "\n"


# ---------------------------------------------------------------------------
# EdaGraph (inc/encode.hpp:18-31), device resident
# ---------------------------------------------------------------------------
class EdaGraph:
    """Learning graph in HBM: symmetric CSR, 4-bit features, labels, fwd_edges."""
    _FREE = "groot_graph_free"


    def __init__(self, handle):
        self._h = handle
        self._free = getattr(lib(), self._FREE)  # bound now: module globals vanish at shutdown

    def __del__(self):
        h, free = getattr(self, "_h", None), getattr(self, "_free", None)
        if h and free is not None:
            free(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def _sizes(self):
        n, nnz, ne = C.c_uint32(), C.c_uint64(), C.c_uint64()
        check(lib().groot_graph_sizes(self._h, C.byref(n), C.byref(nnz), C.byref(ne)))
        return n.value, nnz.value, ne.value

    @property
    def n(self) -> int:
        return self._sizes()[0]

    @property
    def nnz(self) -> int:
        return self._sizes()[1]

    def num_undirected_edges(self) -> int:
        return self._sizes()[2]

    def copy_out(self, *fields):
        n, nnz, ne = self._sizes()
        want = set(fields) or {"row_ptr", "col_idx", "features", "labels", "degree", "fwd_edges"}
        arrs = {
            "row_ptr": np.empty(n + 1, np.uint64) if "row_ptr" in want else None,
            "col_idx": np.empty(nnz, np.uint32) if "col_idx" in want else None,
            "features": np.empty((n, 4), np.uint8) if "features" in want else None,
            "labels": np.empty(n, np.uint8) if "labels" in want else None,
            "degree": np.empty(n, np.uint32) if "degree" in want else None,
            "fwd_edges": np.empty((ne, 2), np.uint32) if "fwd_edges" in want else None,
        }
        check(lib().groot_graph_copy_out(self._h, ptr(arrs["row_ptr"]), ptr(arrs["col_idx"]),
                                         ptr(arrs["features"]), ptr(arrs["labels"]), ptr(arrs["degree"]),
                                         ptr(arrs["fwd_edges"])))
        return {k: v for k, v in arrs.items() if v is not None}

    @property
    def row_ptr(self):
        return self.copy_out("row_ptr")["row_ptr"]

    @property
    def col_idx(self):
        return self.copy_out("col_idx")["col_idx"]

    @property
    def features(self):
        return self.copy_out("features")["features"]

    @property
    def labels(self):
        return self.copy_out("labels")["labels"]

    @property
    def degree(self):
        return self.copy_out("degree")["degree"]

    @property
    def fwd_edges(self):
        return self.copy_out("fwd_edges")["fwd_edges"]

    def device_ptrs(self):
        ps = [C.c_void_p() for _ in range(5)]
        check(lib().groot_graph_device_ptrs(self._h, *[C.byref(p) for p in ps]))
        return dict(zip(["row_ptr", "col_idx", "features", "labels", "fwd_edges"], [p.value for p in ps]))

    @staticmethod
    def from_host(n, row_ptr, col_idx, features=None, labels=None, fwd_edges=None) -> "EdaGraph":
        rp = np.ascontiguousarray(row_ptr, np.uint64)
        ci = np.ascontiguousarray(col_idx, np.uint32)
        ft = None if features is None else np.ascontiguousarray(features, np.uint8)
        lb = None if labels is None else np.ascontiguousarray(labels, np.uint8)
        ed = None if fwd_edges is None else np.ascontiguousarray(fwd_edges, np.uint32)
        h = C.c_void_p()
        check(lib().groot_graph_from_host(n, ptr(rp), ptr(ci), ptr(ft), ptr(lb),
                                          0 if ed is None else ed.shape[0], ptr(ed), C.byref(h)))
        return EdaGraph(h.value)


def encode(aig: Aig, labels=None) -> EdaGraph:
    """src/encode.cpp:33-68: features (K1) + fwd_edges + symmetric CSR (K2) on device."""
    n = aig.num_nodes + int(aig.out_lits.shape[0])
    if labels is not None:
        labels = np.ascontiguousarray(labels, np.uint8)
        if labels.shape[0] != n:
            raise GrootInvalidArgument(1, "encode: label count does not match encoded node count")
    ands = np.ascontiguousarray(aig.and_lits, np.uint32)
    outs = np.ascontiguousarray(aig.out_lits, np.uint32)
    h = C.c_void_p()
    check(lib().groot_encode(aig.num_inputs, aig.num_ands, ptr(ands), int(outs.shape[0]), ptr(outs),
                             ptr(labels), C.byref(h)))
    return EdaGraph(h.value)


def batch(g: EdaGraph, copies: int) -> EdaGraph:
    """src/encode.cpp:70-101 (K3)."""
    h = C.c_void_p()
    check(lib().groot_batch(g.handle, copies, C.byref(h)))
    return EdaGraph(h.value)


# ---------------------------------------------------------------------------
# partition + regrow (inc/partition.hpp)
# ---------------------------------------------------------------------------
class PartitionAssignment:
    _FREE = "groot_assignment_free"

    def __init__(self, handle):
        self._h = handle
        self._free = getattr(lib(), self._FREE)  # bound now: module globals vanish at shutdown

    def __del__(self):
        h, free = getattr(self, "_h", None), getattr(self, "_free", None)
        if h and free is not None:
            free(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def k(self) -> int:
        n, k = C.c_uint32(), C.c_uint32()
        check(lib().groot_assignment_info(self._h, C.byref(n), C.byref(k)))
        return k.value

    @property
    def part_of(self) -> np.ndarray:
        n, k = C.c_uint32(), C.c_uint32()
        check(lib().groot_assignment_info(self._h, C.byref(n), C.byref(k)))
        out = np.empty(n.value, np.uint32)
        check(lib().groot_assignment_copy_out(self._h, ptr(out)))
        return out

    @staticmethod
    def from_host(part_of) -> "PartitionAssignment":
        p = np.ascontiguousarray(part_of, np.uint32)
        h = C.c_void_p()
        check(lib().groot_assignment_from_host(p.shape[0], ptr(p), C.byref(h)))
        return PartitionAssignment(h.value)


def partition_topo_chunks(g: EdaGraph, k: int) -> PartitionAssignment:
    """src/partition.cpp:301-312 (K4)."""
    h = C.c_void_p()
    check(lib().groot_partition_topo_chunks(g.handle, k, C.byref(h)))
    return PartitionAssignment(h.value)


def partition_multilevel(g: EdaGraph, k: int, seed: int = 7, stats: dict | None = None) -> PartitionAssignment:
    """src/partition.cpp:314-367 replacement: topo chunks + device label propagation
    within the 5 % balance cap; terminates for every k. `stats` (optional dict)
    receives the rounds run and nodes moved."""
    h = C.c_void_p()
    rounds, moves = C.c_uint32(), C.c_uint64()
    check(lib().groot_partition_multilevel(g.handle, k, seed, C.byref(h), C.byref(rounds), C.byref(moves)))
    if stats is not None:
        stats.update(rounds=rounds.value, moves=moves.value)
    return PartitionAssignment(h.value)


def load_assignment(path: str, n: int) -> PartitionAssignment:
    """src/partition.cpp:369-392."""
    h = C.c_void_p()
    check(lib().groot_load_assignment(path.encode(), n, C.byref(h)))
    return PartitionAssignment(h.value)


def save_assignment(path: str, pa: PartitionAssignment):
    """src/partition.cpp:394-398."""
    with open(path, "w") as f:
        f.writelines(f"{v} {p}\n" for v, p in enumerate(pa.part_of.tolist()))


def crossing_fraction(g: EdaGraph, pa: PartitionAssignment) -> float:
    out = C.c_double()
    check(lib().groot_crossing_fraction(g.handle, pa.handle, C.byref(out)))
    return out.value


def edge_cut(g: EdaGraph, pa: PartitionAssignment) -> int:
    out = C.c_uint64()
    check(lib().groot_edge_cut(g.handle, pa.handle, C.byref(out)))
    return out.value


@dataclass
class AugmentedPartition:
    """inc/partition.hpp:23-33 (host copy of one part)."""
    core_nodes: np.ndarray
    boundary_nodes: np.ndarray
    edges: np.ndarray

    @property
    def local_to_global(self):
        return np.concatenate([self.core_nodes, self.boundary_nodes])

    @property
    def core_mask(self):
        m = np.zeros(self.core_nodes.shape[0] + self.boundary_nodes.shape[0], np.uint8)
        m[: self.core_nodes.shape[0]] = 1
        return m

    @property
    def local_index(self):
        return {int(v): i for i, v in enumerate(self.local_to_global.tolist())}

    def num_core(self):
        return int(self.core_nodes.shape[0])

    def size(self):
        return int(self.core_nodes.shape[0] + self.boundary_nodes.shape[0])


class AugmentedPartitions:
    """vector<AugmentedPartition> living in HBM (result of regrow/core_subgraphs)."""
    _FREE = "groot_parts_free"


    def __init__(self, handle):
        self._h = handle
        self._free = getattr(lib(), self._FREE)  # bound now: module globals vanish at shutdown

    def __del__(self):
        h, free = getattr(self, "_h", None), getattr(self, "_free", None)
        if h and free is not None:
            free(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def __len__(self):
        k = C.c_uint32()
        check(lib().groot_parts_count(self._h, C.byref(k)))
        return k.value

    def sizes(self, p):
        nc, nb, ne = C.c_uint32(), C.c_uint32(), C.c_uint64()
        check(lib().groot_parts_sizes(self._h, p, C.byref(nc), C.byref(nb), C.byref(ne)))
        return nc.value, nb.value, ne.value

    def __getitem__(self, p) -> AugmentedPartition:
        if p < 0:
            p += len(self)
        nc, nb, ne = self.sizes(p)
        core = np.empty(nc, np.uint32)
        bnd = np.empty(nb, np.uint32)
        edges = np.empty((ne, 2), np.uint32)
        check(lib().groot_parts_copy_out(self._h, p, ptr(core), ptr(bnd), ptr(edges)))
        return AugmentedPartition(core, bnd, edges)

    def __iter__(self):
        return (self[p] for p in range(len(self)))

    @staticmethod
    def from_host(n: int, parts) -> "AugmentedPartitions":
        """Upload a list of AugmentedPartition as given (groot_parts_from_host)."""
        parts = list(parts)
        k = len(parts)
        cores = [np.ascontiguousarray(p.core_nodes, np.uint32) for p in parts]
        bnds = [np.ascontiguousarray(p.boundary_nodes, np.uint32) for p in parts]
        edges = [np.ascontiguousarray(p.edges, np.uint32).reshape(-1, 2) for p in parts]
        off = lambda arrs: np.concatenate([[0], np.cumsum([a.shape[0] for a in arrs])]).astype(np.uint64)
        cat = lambda arrs: np.ascontiguousarray(np.concatenate(arrs) if arrs else np.zeros(0, np.uint32), np.uint32)
        # (keep every array referenced until the call returns: ptr() holds no reference)
        co, ca, bo, ba = off(cores), cat(cores), off(bnds), cat(bnds)
        eo, ea = off(edges), cat([e.ravel() for e in edges])
        h = C.c_void_p()
        check(lib().groot_parts_from_host(n, k, ptr(co), ptr(ca), ptr(bo), ptr(ba), ptr(eo), ptr(ea), C.byref(h)))
        return AugmentedPartitions(h.value)


def regrow(g: EdaGraph, pa: PartitionAssignment) -> AugmentedPartitions:
    """Algorithm 1 boundary re-growth (src/partition.cpp:460-462; K5, K6)."""
    h = C.c_void_p()
    check(lib().groot_regrow(g.handle, pa.handle, 1, C.byref(h)))
    return AugmentedPartitions(h.value)


def core_subgraphs(g: EdaGraph, pa: PartitionAssignment) -> AugmentedPartitions:
    """Ablation without boundary nodes (src/partition.cpp:464-466)."""
    h = C.c_void_p()
    check(lib().groot_regrow(g.handle, pa.handle, 0, C.byref(h)))
    return AugmentedPartitions(h.value)


def footprint_proxy(parts: AugmentedPartitions, feature_cols: int = 4, hidden_dim: int = 32) -> int:
    out = C.c_uint64()
    check(lib().groot_footprint_proxy(parts.handle, feature_cols, hidden_dim, C.byref(out)))
    return out.value


def materialize(g: EdaGraph, parts: AugmentedPartitions, p: int) -> EdaGraph:
    """src/partition.cpp:488-506 (K7)."""
    h = C.c_void_p()
    check(lib().groot_materialize(g.handle, parts.handle, p, C.byref(h)))
    return EdaGraph(h.value)


# ---------------------------------------------------------------------------
# model + forward + classify (inc/gnn.hpp)
# ---------------------------------------------------------------------------
def param_count(depth=4, in_dim=4, hidden=32, classes=NUM_CLASSES) -> int:
    return int(lib().groot_param_count(depth, in_dim, hidden, classes))


class Model:
    """Model (inc/gnn.hpp:26-33) resident on the device (weights split TF32 hi/lo)."""
    _FREE = "groot_model_free"


    def __init__(self, handle):
        self._h = handle
        self._free = getattr(lib(), self._FREE)  # bound now: module globals vanish at shutdown

    def __del__(self):
        h, free = getattr(self, "_h", None), getattr(self, "_free", None)
        if h and free is not None:
            free(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def info(self):
        d, i, h, c = (C.c_uint32() for _ in range(4))
        check(lib().groot_model_info(self._h, C.byref(d), C.byref(i), C.byref(h), C.byref(c)))
        return dict(depth=d.value, in_dim=i.value, hidden=h.value, classes=c.value)

    @property
    def params(self) -> np.ndarray:
        inf = self.info()
        out = np.empty(param_count(**inf), np.float64)
        check(lib().groot_model_params(self._h, ptr(out)))
        return out

    @staticmethod
    def from_params(params, depth=4, in_dim=4, hidden=32, classes=NUM_CLASSES) -> "Model":
        prm = np.ascontiguousarray(params, np.float64)
        if prm.shape[0] != param_count(depth, in_dim, hidden, classes):
            raise GrootInvalidArgument(1, "model: parameter count does not match the shape")
        h = C.c_void_p()
        check(lib().groot_model_create(depth, in_dim, hidden, classes, ptr(prm), C.byref(h)))
        return Model(h.value)


def init_params(seed: int, in_dim=4, hidden=32, classes=NUM_CLASSES, depth=4) -> np.ndarray:
    out = np.empty(param_count(depth, in_dim, hidden, classes), np.float64)
    check(lib().groot_init_params(seed, in_dim, hidden, classes, depth, ptr(out)))
    return out


def init_model(seed: int, in_dim=4, hidden=32, num_classes=NUM_CLASSES, depth=4) -> Model:
    """src/gnn.cpp:113-138 (mt19937_64 Glorot; bit-identical weights)."""
    return Model.from_params(init_params(seed, in_dim, hidden, num_classes, depth), depth, in_dim, hidden,
                             num_classes)


def load_model(path: str) -> Model:
    """src/gnn.cpp:349-372 (ASG1)."""
    h = C.c_void_p()
    check(lib().groot_model_load(path.encode(), C.byref(h)))
    return Model(h.value)


def save_model(path: str, model: Model):
    check(lib().groot_model_save(model.handle, path.encode()))


@dataclass
class TrainStats:
    """inc/gnn.hpp:47-50: per-epoch loss and training accuracy."""
    loss: np.ndarray
    accuracy: np.ndarray


def train(g: EdaGraph, epochs: int = 100, learning_rate: float = 1e-3, seed: int = 7, beta1: float = 0.9,
          beta2: float = 0.999, adam_eps: float = 1e-8, depth: int = 4, hidden: int = 32,
          classes: int = NUM_CLASSES, init=None, stats: TrainStats | None = None) -> Model:
    """train (src/gnn.cpp:211-255) on the device, fp64: full-batch Adam from
    init_model(seed) (or `init`, a parameter vector in ASG1 order)."""
    np_ = param_count(depth, 4, hidden, classes)
    out = np.empty(np_, np.float64)
    loss = np.empty(max(epochs, 1), np.float64)
    acc = np.empty(max(epochs, 1), np.float64)
    ini = None if init is None else np.ascontiguousarray(init, np.float64)
    check(lib().groot_train(g.handle, depth, 4, hidden, classes, epochs, learning_rate, seed, beta1, beta2, adam_eps,
                            ptr(ini), ptr(out), ptr(loss), ptr(acc)))
    if stats is not None:
        stats.loss, stats.accuracy = loss[:epochs], acc[:epochs]
    return Model.from_params(out, depth, 4, hidden, classes)


def loss_and_grads(params, g: EdaGraph, depth: int = 4, hidden: int = 32, classes: int = NUM_CLASSES):
    """loss_and_grads (src/gnn.cpp:180-209) on the device: (loss, grads in ASG1 order)."""
    prm = np.ascontiguousarray(params, np.float64)
    grads = np.empty_like(prm)
    loss = C.c_double()
    check(lib().groot_loss_and_grads(g.handle, depth, 4, hidden, classes, ptr(prm), ptr(grads), C.byref(loss)))
    return loss.value, grads


def grad_check(params, g: EdaGraph, epsilon: float = 1e-4, depth: int = 4, hidden: int = 32,
               classes: int = NUM_CLASSES) -> float:
    """grad_check (inc/gnn.hpp:88-90): max over parameters of |a - n| / max(|a|, |n|, 1),
    analytic (device backward) vs central differences (device forward losses)."""
    prm = np.ascontiguousarray(params, np.float64)
    _, ana = loss_and_grads(prm, g, depth, hidden, classes)
    worst = 0.0
    for i in range(prm.shape[0]):
        p = prm.copy()
        p[i] += epsilon
        lp, _ = loss_and_grads(p, g, depth, hidden, classes)
        p[i] -= 2 * epsilon
        lm, _ = loss_and_grads(p, g, depth, hidden, classes)
        num = (lp - lm) / (2 * epsilon)
        worst = max(worst, abs(ana[i] - num) / max(abs(ana[i]), abs(num), 1.0))
    return worst


@dataclass
class Prediction:
    """inc/gnn.hpp:75-79."""
    labels: np.ndarray
    confusion: np.ndarray
    accuracy: float


def forward(model: Model, g) -> np.ndarray:
    """src/gnn.cpp:172-178: n x classes logits (fp32 on device). g: EdaGraph or SageContext."""
    if isinstance(g, SageContext):
        g = g.graph
    c = model.info()["classes"]
    out = np.empty((g.n, c), np.float32)
    check(lib().groot_forward(model.handle, g.handle, ptr(out)))
    return out


class SageContext:
    """make_context (src/gnn.cpp:140-170): the per-graph state the forward derives
    from the graph alone (row classifier, tile plan, HD plan, activation buffers),
    built on the device and cached on the resident graph. forward(model, ctx)
    reuses it; release() frees it."""

    def __init__(self, g: EdaGraph):
        self.graph = g
        check(lib().groot_graph_prepare(g.handle))

    @property
    def labels(self):
        return self.graph.labels

    def release(self):
        check(lib().groot_graph_release_context(self.graph.handle))


def make_context(g: EdaGraph) -> SageContext:
    return SageContext(g)


def layer_dev(model: Model, g: EdaGraph, layer: int, hin=None, hout=None, labels=None, logits=None):
    """One layer of run_forward (src/gnn.cpp:37-52) on device tensors (torch),
    enqueued on the library stream: layer 0 reads the node features; the last
    layer writes labels (u8[n]) and optionally logits. See groot_layer_dev."""
    def dp(t):
        return None if t is None else C.c_void_p(t.data_ptr())
    check(lib().groot_layer_dev(model.handle, g.handle, layer, dp(hin), dp(hout), dp(labels), dp(logits)))


def forward_naive(model: Model, g: EdaGraph):
    """Differential-test path (thread-per-row kernels). Returns (logits, labels)."""
    c = model.info()["classes"]
    n = g.n
    lg = np.empty((n, c), np.float32)
    lab = np.empty(n, np.uint8)
    check(lib().groot_debug_forward_naive(model.handle, g.handle, ptr(lg), ptr(lab)))
    return lg, lab


def predict_full(model: Model, g) -> Prediction:
    """src/gnn.cpp:293-300. g: EdaGraph or SageContext."""
    if isinstance(g, SageContext):
        g = g.graph
    n = g.n
    labels = np.empty(n, np.uint8)
    conf = np.zeros((5, 5), np.uint64)
    acc = C.c_double()
    check(lib().groot_predict_full(model.handle, g.handle, ptr(labels), ptr(conf), C.byref(acc)))
    return Prediction(labels, conf, acc.value)


def predict(model: Model, g: EdaGraph, parts) -> Prediction:
    """src/gnn.cpp:280-291: every node scored from its core partition. `parts` is a
    device AugmentedPartitions (regrow's result) or a list of AugmentedPartition."""
    n = g.n
    if not isinstance(parts, AugmentedPartitions):
        parts = AugmentedPartitions.from_host(n, parts)
    labels = np.empty(n, np.uint8)
    conf = np.zeros((5, 5), np.uint64)
    acc = C.c_double()
    check(lib().groot_predict(model.handle, g.handle, parts.handle, ptr(labels), ptr(conf), C.byref(acc)))
    return Prediction(labels, conf, acc.value)


def predict_parts(model: Model, g: EdaGraph, parts: AugmentedPartitions, part_ids, labels=None) -> np.ndarray:
    """predict restricted to `part_ids`: returns the global label vector with the core
    nodes of those parts filled in (others from `labels`, default zeros)."""
    ids = np.ascontiguousarray(part_ids, np.uint32)
    out = np.zeros(g.n, np.uint8) if labels is None else np.ascontiguousarray(labels, np.uint8).copy()
    check(lib().groot_predict_parts(model.handle, g.handle, parts.handle, ptr(ids), ids.shape[0], ptr(out)))
    return out


def classify_aig(model: Model, aig: Aig, labels, copies: int = 1) -> Prediction:
    """End to end: host AIG -> encode -> batch -> predict_full -> host classes."""
    ands = np.ascontiguousarray(aig.and_lits, np.uint32)
    outs = np.ascontiguousarray(aig.out_lits, np.uint32)
    lab = None if labels is None else np.ascontiguousarray(labels, np.uint8)
    n = (aig.num_nodes + outs.shape[0]) * copies
    pred = np.empty(n, np.uint8)
    conf = np.zeros((5, 5), np.uint64)
    acc = C.c_double()
    check(lib().groot_classify_aig(model.handle, aig.num_inputs, aig.num_ands, ptr(ands), outs.shape[0],
                                   ptr(outs), ptr(lab), copies, ptr(pred), ptr(conf), C.byref(acc)))
    return Prediction(pred, conf, acc.value)


# ---------------------------------------------------------------------------
# verification consumer of the classes (inc/verify.hpp, src/verify.cpp)
# ---------------------------------------------------------------------------
@dataclass
class VerifyReport:
    """inc/verify.hpp:19-27 (the residual as text, first 64 terms)."""
    equivalent: bool
    inconclusive: bool
    residual_terms: int
    residual: str
    substitution_count: int
    shortcut_count: int
    fallback_count: int


def backward_rewrite(aig: Aig, labels, width: int, supports: dict | None = None,
                     monomial_cap: int = 2_000_000) -> VerifyReport:
    """src/verify.cpp:220-395: label-guided backward rewriting (host, BigInt)."""
    ands = np.ascontiguousarray(aig.and_lits, np.uint32)
    outs = np.ascontiguousarray(aig.out_lits, np.uint32)
    lab = np.ascontiguousarray(labels, np.uint8)
    off = nodes = None
    if supports:
        nn = aig.num_nodes
        cnt = np.zeros(nn, np.uint32)
        for v, sup in supports.items():
            if v < nn:
                cnt[v] = len(sup)
        off = np.concatenate([[0], np.cumsum(cnt)]).astype(np.uint32)
        nodes = np.zeros(int(off[-1]), np.uint32)
        for v, sup in supports.items():
            if v < nn:
                nodes[off[v]:off[v + 1]] = [x >> 1 for x in sup]
    eq, inc = C.c_int32(), C.c_int32()
    rt = C.c_uint64()
    counts = np.zeros(3, np.uint64)
    check(lib().groot_backward_rewrite(aig.num_inputs, aig.num_ands, ptr(ands), outs.shape[0], ptr(outs), ptr(lab),
                                       lab.shape[0], ptr(off), ptr(nodes), width, monomial_cap, C.byref(eq),
                                       C.byref(inc), C.byref(rt), ptr(counts)))
    return VerifyReport(bool(eq.value), bool(inc.value), rt.value, lib().groot_backward_rewrite_residual().decode(),
                        int(counts[0]), int(counts[1]), int(counts[2]))


def truth_table_equiv(aig: Aig, width: int) -> bool:
    """src/verify.cpp:398-416 (2*width <= 20)."""
    ands = np.ascontiguousarray(aig.and_lits, np.uint32)
    outs = np.ascontiguousarray(aig.out_lits, np.uint32)
    eq = C.c_int32()
    check(lib().groot_truth_table_equiv(aig.num_inputs, aig.num_ands, ptr(ands), outs.shape[0], ptr(outs), width,
                                        C.byref(eq)))
    return bool(eq.value)


def simulate(aig: Aig, inputs) -> np.ndarray:
    """src/aig.cpp:130-138: output bits for one input assignment."""
    ands = np.ascontiguousarray(aig.and_lits, np.uint32)
    outs = np.ascontiguousarray(aig.out_lits, np.uint32)
    inp = np.ascontiguousarray(inputs, np.uint8)
    if inp.shape[0] != aig.num_inputs:
        raise GrootInvalidArgument(1, "simulate: assignment length != number of inputs")
    out = np.empty(outs.shape[0], np.uint8)
    check(lib().groot_simulate(aig.num_inputs, aig.num_ands, ptr(ands), outs.shape[0], ptr(outs), ptr(inp), ptr(out)))
    return out


# ---------------------------------------------------------------------------
# spmm (inc/spmm.hpp)
# ---------------------------------------------------------------------------
def build_plan(g: EdaGraph, hd_threshold=512, ld_threshold=12, nz_budget=96) -> dict:
    """src/spmm.cpp:37-127 — the reference SpmmPlan (degree sort on device)."""
    counts = np.zeros(6, np.uint64)
    check(lib().groot_build_plan(g.handle, hd_threshold, ld_threshold, nz_budget, ptr(counts),
                                 None, None, None, None, None))
    n = g.n
    perm = np.empty(n, np.uint32)
    hd = np.empty(int(counts[0]), np.uint32)
    mid = np.empty(int(counts[1]), np.uint32)
    ldg = np.empty((int(counts[2]), 3), np.uint32)
    units = np.empty((int(counts[3]), 6), np.uint64)
    check(lib().groot_build_plan(g.handle, hd_threshold, ld_threshold, nz_budget, ptr(counts), ptr(perm),
                                 ptr(hd), ptr(mid), ptr(ldg), ptr(units)))
    return {"perm": perm, "hd_rows": hd, "mid_rows": mid, "ld_groups": ldg, "units": units,
            "ld_row_begin": int(counts[4]), "ld_row_end": int(counts[5])}


def build_plan_rows(row_ptr, hd_threshold=512, ld_threshold=12, nz_budget=96) -> dict:
    """build_plan(rows, span row_ptr, ...) (src/spmm.cpp:37-127) from a host row_ptr."""
    rp = np.ascontiguousarray(row_ptr, np.uint64)
    rows = rp.shape[0] - 1
    counts = np.zeros(6, np.uint64)
    check(lib().groot_build_plan_rows(rows, ptr(rp), hd_threshold, ld_threshold, nz_budget, ptr(counts),
                                      None, None, None, None, None))
    perm = np.empty(rows, np.uint32)
    hd = np.empty(int(counts[0]), np.uint32)
    mid = np.empty(int(counts[1]), np.uint32)
    ldg = np.empty((int(counts[2]), 3), np.uint32)
    units = np.empty((int(counts[3]), 6), np.uint64)
    check(lib().groot_build_plan_rows(rows, ptr(rp), hd_threshold, ld_threshold, nz_budget, ptr(counts), ptr(perm),
                                      ptr(hd), ptr(mid), ptr(ldg), ptr(units)))
    return {"perm": perm, "hd_rows": hd, "mid_rows": mid, "ld_groups": ldg, "units": units,
            "ld_row_begin": int(counts[4]), "ld_row_end": int(counts[5]), "rows": rows, "nnz": int(rp[-1])}


def degree_sort(row_ptr):
    """src/spmm.cpp:9-35: (perm, sorted_row_ptr)."""
    rp = np.ascontiguousarray(row_ptr, np.uint64)
    rows = rp.shape[0] - 1
    perm = np.empty(rows, np.uint32)
    srp = np.empty(rows + 1, np.uint64)
    check(lib().groot_degree_sort(rows, ptr(rp), ptr(perm), ptr(srp)))
    return perm, srp


def spmm_csr_f64(row_ptr, col_idx, values, dense, cols=None, hd_threshold=512) -> np.ndarray:
    """spmm::execute over CsrMatrix<double> on the device, bitwise the reference's
    execute with a plan of this hd_threshold (0: reference_spmm's row loop)."""
    rp = np.ascontiguousarray(row_ptr, np.uint64)
    ci = np.ascontiguousarray(col_idx, np.uint32)
    vals = None if values is None else np.ascontiguousarray(values, np.float64)
    d = np.ascontiguousarray(dense, np.float64)
    rows = rp.shape[0] - 1
    cols = d.shape[0] if cols is None else cols
    if d.shape[0] != cols:
        raise GrootInvalidArgument(1, "spmm::execute: dense shape mismatch")
    out = np.empty((rows, d.shape[1]), np.float64)
    check(lib().groot_spmm_csr_f64(rows, cols, ptr(rp), ptr(ci), ptr(vals), ptr(d), d.shape[1], hd_threshold,
                                   ptr(out)))
    return out


def spmm_mean(g: EdaGraph, dense: np.ndarray) -> np.ndarray:
    """out = D^-1 A dense (spmm::execute over make_context's a_mean), fp32."""
    d = np.ascontiguousarray(dense, np.float32)
    if d.shape[0] != g.n:
        raise GrootInvalidArgument(1, "spmm::execute: dense shape mismatch")
    out = np.empty_like(d)
    check(lib().groot_spmm_mean(g.handle, ptr(d), d.shape[1], ptr(out)))
    return out


def spmm_csr(row_ptr, col_idx, values, dense, cols=None, hd_threshold=512) -> np.ndarray:
    """spmm::execute over a general CsrMatrix<float> (inc/spmm.hpp:106-181); see spmm_csr_f64."""
    rp = np.ascontiguousarray(row_ptr, np.uint64)
    ci = np.ascontiguousarray(col_idx, np.uint32)
    vals = None if values is None else np.ascontiguousarray(values, np.float32)
    d = np.ascontiguousarray(dense, np.float32)
    rows = rp.shape[0] - 1
    cols = d.shape[0] if cols is None else cols
    if d.shape[0] != cols:
        raise GrootInvalidArgument(1, "spmm::execute: dense shape mismatch")
    out = np.empty((rows, d.shape[1]), np.float32)
    check(lib().groot_spmm_csr(rows, cols, ptr(rp), ptr(ci), ptr(vals), ptr(d), d.shape[1], hd_threshold, ptr(out)))
    return out


def kernel_launches() -> int:
    return int(lib().groot_kernel_launches())


def set_stream(stream_ptr: int | None):
    check(lib().groot_set_stream(stream_ptr))
