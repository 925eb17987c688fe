"""Data-parallel sharding of the hot path over ranks (one process per GPU).

The path shards naturally:

* **Batch copies.** ``batch(g, b)`` is b disjoint copies of one circuit. Rank r
  of G owns a contiguous run of copies; node i of copy k is global id k*n1+i, so
  a rank's shard is itself ``batch(g1, count)`` shifted by ``first*n1``. No
  feature exchange is needed in the data path.
* **Partitions.** For partitioned inference (``predict`` over regrown parts,
  src/gnn.cpp:280-291) each part is forwarded independently — the reference
  never exchanges features between parts — so parts are dealt
  round-robin to ranks.

The only collectives are the assembly of global results: an integer
all-reduce of the 5x5 confusion counts (exact, order-independent) and, when a
caller wants the global label vector on every rank, an all-gather of the
per-rank label blocks. Both go through ``torch.distributed`` (NCCL on the
GPU box, gloo in the CPU tests).

The compute callables are injected so the same host logic runs over the
device path (default) or over the CPU oracle in tests.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np


@dataclass(frozen=True)
class CopyShard:
    first: int      # first batch copy owned by this rank
    count: int      # number of copies
    node_offset: int
    nodes: int


def copy_shard(rank: int, world: int, copies: int, n1: int) -> CopyShard:
    """Balanced contiguous split of `copies` batch copies over `world` ranks."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard: bad rank/world")
    if copies < world:
        raise ValueError("shard: fewer batch copies than ranks (use partition sharding)")
    first = copies * rank // world
    last = copies * (rank + 1) // world
    return CopyShard(first, last - first, first * n1, (last - first) * n1)


def owned_parts(k: int, rank: int, world: int) -> list[int]:
    """Round-robin ownership of k partitions."""
    return list(range(rank, k, world))


def _dist():
    import torch.distributed as dist
    return dist


def allreduce_confusion(conf: np.ndarray, device=None) -> np.ndarray:
    """Exact integer all-reduce of the 5x5 confusion counts."""
    import torch
    t = torch.as_tensor(np.asarray(conf, dtype=np.int64).reshape(-1), device=device)
    _dist().all_reduce(t)
    return t.cpu().numpy().astype(np.uint64).reshape(5, 5)


def allgather_blocks(block: np.ndarray, device=None) -> list[np.ndarray]:
    """All-gather variable-length u8 blocks (one per rank), rank order."""
    import torch
    dist = _dist()
    world = dist.get_world_size()
    n = torch.tensor([block.shape[0]], dtype=torch.int64, device=device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    cap = int(max(int(s.item()) for s in sizes))
    buf = torch.zeros(cap, dtype=torch.uint8, device=device)
    buf[: block.shape[0]] = torch.as_tensor(block, dtype=torch.uint8, device=device)
    outs = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf)
    return [o[: int(s.item())].cpu().numpy() for o, s in zip(outs, sizes)]


def predict_copies(rank: int, world: int, copies: int, n1: int,
                   compute: Callable[[CopyShard], tuple[np.ndarray, np.ndarray]],
                   gather: bool = True, device=None):
    """Sharded predict_full over batch copies.

    compute(shard) -> (labels u8[shard.nodes], confusion 5x5) for the rank's copies.
    Returns (global labels or None, global confusion, accuracy)."""
    shard = copy_shard(rank, world, copies, n1)
    labels, conf = compute(shard)
    gconf = allreduce_confusion(conf, device) if world > 1 else np.asarray(conf, np.uint64)
    total = copies * n1
    acc = float(np.trace(gconf)) / total if total else 0.0
    glabels = None
    if gather:
        glabels = np.concatenate(allgather_blocks(labels, device)) if world > 1 else labels
    return glabels, gconf, acc


def predict_parts(rank: int, world: int, k: int, n: int, truth: np.ndarray,
                  compute: Callable[[Sequence[int]], tuple[np.ndarray, np.ndarray]],
                  device=None):
    """Sharded predict over k regrown partitions.

    compute(part_ids) -> (core global ids u32[m], labels u8[m]) for the rank's parts.
    Returns (global labels, confusion, accuracy) on every rank."""
    ids, lab = compute(owned_parts(k, rank, world))
    ids = np.asarray(ids, np.uint32)
    lab = np.asarray(lab, np.uint8)
    if world > 1:
        id_blocks = allgather_blocks(ids.view(np.uint8), device)
        lab_blocks = allgather_blocks(lab, device)
        ids = np.concatenate([b.view(np.uint32) for b in id_blocks])
        lab = np.concatenate(lab_blocks)
    pred = np.zeros(n, np.uint8)
    pred[ids] = lab
    conf = np.zeros((5, 5), np.uint64)
    np.add.at(conf, (truth.astype(np.int64), pred.astype(np.int64)), 1)
    acc = float((pred == truth).sum()) / n if n else 0.0
    return pred, conf, acc


# ---------------------------------------------------------------------------
# device-path compute functions (GPU box)
# ---------------------------------------------------------------------------
def device_copy_compute(model, circuit):
    """compute(shard) over the device path: encode one copy, batch `count`, predict_full."""
    from . import api

    def compute(shard: CopyShard):
        g1 = api.encode(circuit.aig, circuit.labels)
        g = api.batch(g1, shard.count) if shard.count > 1 else g1
        p = api.predict_full(model, g)
        return p.labels, p.confusion
    return compute


def device_parts_compute(model, graph, parts):
    """compute(part_ids) over the device path: predict on the union of the rank's parts."""
    from . import api

    def compute(part_ids: Sequence[int]):
        labels = api.predict_parts(model, graph, parts, list(part_ids))  # only this rank's parts
        ids = np.concatenate([parts[p].core_nodes for p in part_ids]) if part_ids else np.zeros(0, np.uint32)
        return ids, labels[ids]
    return compute


# ---------------------------------------------------------------------------
# Exact-halo mode X: whole-graph (predict_full) results for
# partitions that straddle ranks. Rank r owns part r of a k = world partition
# and forwards the materialized regrown part (cores first, then the 1-hop
# boundary, src/partition.cpp:428-438 local ids). Every core row has its full
# neighbour list there, so a layer is exact on core rows once the boundary
# rows hold their owners' values of the previous layer: after each layer but
# the last, every rank sends the core rows its peers have as boundary rows
# (one all-to-all per layer; NCCL over NVLink on the box). Boundary rows'
# own outputs are partial and are overwritten by the exchange. Contrast mode
# R (predict_parts above, the reference's semantics): no exchange, boundary
# rows keep their partial neighbourhoods through every layer.
# ---------------------------------------------------------------------------
@dataclass
class HaloPlan:
    """One rank's exchange plan. send[q]: local core indices rank q needs, in
    ascending global order; recv[q]: local boundary indices that rank q's rows
    fill, in the same order."""
    rank: int
    world: int
    num_core: int
    num_local: int
    core_nodes: np.ndarray
    send: list
    recv: list

    @property
    def send_counts(self):
        return [int(x.shape[0]) for x in self.send]

    @property
    def recv_counts(self):
        return [int(x.shape[0]) for x in self.recv]


def halo_plans(part_of: np.ndarray, cores: Sequence[np.ndarray], boundaries: Sequence[np.ndarray]) -> list:
    """Exchange plans of all k ranks from the regrown parts (core_nodes and
    boundary_nodes, both ascending global ids, as regrow returns them)."""
    k = len(cores)
    part_of = np.asarray(part_of)
    plans = []
    for r in range(k):
        core_r = np.asarray(cores[r], np.int64)
        bnd_r = np.asarray(boundaries[r], np.int64)
        owner = part_of[bnd_r] if bnd_r.size else np.zeros(0, np.int64)
        recv = [core_r.shape[0] + np.nonzero(owner == q)[0] for q in range(k)]
        send = []
        for q in range(k):
            bq = np.asarray(boundaries[q], np.int64)
            mine = bq[part_of[bq] == r] if bq.size else bq
            send.append(np.searchsorted(core_r, mine))
        plans.append(HaloPlan(r, k, core_r.shape[0], core_r.shape[0] + bnd_r.shape[0], core_r, send, recv))
    for r in range(k):  # every row sent is a core row of its sender, in the receiver's order
        for q in range(k):
            assert plans[r].send[q].shape == plans[q].recv[r].shape
    return plans


class HaloExchanger:
    """Device-resident exchange of one rank's boundary rows (mode X).

    The plan's index lists are uploaded once (send rows gathered by one
    index_select, received rows scattered by one index_copy_) and the send /
    receive buffers are allocated once for the row width; each call is then
    gather -> all_to_all_single (NCCL over NVLink on the box) -> scatter with
    no host work and no host<->device copy."""

    def __init__(self, plan: HaloPlan, f: int, device, dtype=None):
        import torch
        self.plan = plan
        dtype = dtype or torch.float32
        send = np.concatenate(plan.send) if plan.send else np.zeros(0, np.int64)
        recv = np.concatenate(plan.recv) if plan.recv else np.zeros(0, np.int64)
        self.send_idx = torch.as_tensor(send.astype(np.int64), device=device)
        self.recv_idx = torch.as_tensor(recv.astype(np.int64), device=device)
        self.send_buf = torch.empty((self.send_idx.shape[0], f), dtype=dtype, device=device)
        self.recv_buf = torch.empty((self.recv_idx.shape[0], f), dtype=dtype, device=device)
        self.send_counts = plan.send_counts
        self.recv_counts = plan.recv_counts
        self.bytes_per_call = int(self.send_buf.numel() + self.recv_buf.numel()) * self.send_buf.element_size()

    def __call__(self, h, plan=None):
        import torch
        torch.index_select(h, 0, self.send_idx, out=self.send_buf)
        _dist().all_to_all_single(self.recv_buf, self.send_buf, self.recv_counts, self.send_counts)
        h.index_copy_(0, self.recv_idx, self.recv_buf)
        return h


def exchange_halo(h, plan: HaloPlan):
    """One-shot all-to-all of the boundary rows of a (num_local x f) torch tensor,
    in place (builds a HaloExchanger; reuse one across layers instead)."""
    return HaloExchanger(plan, h.shape[1], h.device, h.dtype)(h)


def predict_exact(plan: HaloPlan, depth: int, layer: Callable, exchange: Callable = exchange_halo):
    """Mode-X forward of one rank: layer(l, h_in) -> h_out (num_local x hidden),
    or for the last layer the (num_local x classes) logits; exchange after every
    layer but the last. Returns the logits of the rank's core rows."""
    h = None
    for l in range(depth):
        h = layer(l, h)
        if l + 1 < depth:
            h = exchange(h, plan)
    return h[: plan.num_core]


def device_layer_fn(model, local_graph, hidden: int = 32):
    """layer(l, h) over the device path (groot_layer_dev) on a rank's local graph."""
    import torch
    from . import api
    n = local_graph.n
    info = model.info()

    def layer(l, h):
        if l + 1 < info["depth"]:
            out = torch.empty((n, hidden), dtype=torch.float32, device="cuda")
            api.layer_dev(model, local_graph, l, h, out, None, None)
            return out
        cls = torch.empty(n, dtype=torch.uint8, device="cuda")
        logits = torch.empty((n, info["classes"]), dtype=torch.float32, device="cuda")
        api.layer_dev(model, local_graph, l, h, None, cls, logits)
        return logits
    return layer
