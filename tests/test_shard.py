"""Multi-rank sharding logic (paper_2511_18297_b200/shard.py) with world_size 2 over
gloo on CPU. The per-rank compute is the oracle (the device path on the GPU box
is covered by test_gpu_parity / test_shard_device); results must equal the
single-process reference prediction exactly."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import pyoracle as O
from paper_2511_18297_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        prm = O.init_model(7)
        g1 = O.encode(O.gen_csa(8))
        if mode == "copies":
            copies = 5

            def compute(sh):
                g = O.batch(g1, sh.count) if sh.count > 1 else g1
                pred, conf, _, _ = O.predict_full(g, prm)
                return pred, conf
            labels, conf, acc = shard.predict_copies(rank, world, copies, g1.n, compute)
            np.savez(os.path.join(out_dir, f"r{rank}.npz"), labels=labels, conf=conf, acc=acc)
        else:
            g = O.batch(g1, 2)
            k = 5
            parts = O.regrow(g, O.topo_chunks(g.n, k), k)

            def compute(ids):
                core, lab = [], []
                for p in ids:
                    sub = O.materialize(g, parts[p])
                    pp, _, _ = O.classify(O.forward(sub, prm))
                    core.append(parts[p].core_nodes)
                    lab.append(pp[: parts[p].num_core])
                if not core:
                    return np.zeros(0, np.uint32), np.zeros(0, np.uint8)
                return np.concatenate(core), np.concatenate(lab)
            labels, conf, acc = shard.predict_parts(rank, world, k, g.n, g.labels, compute)
            np.savez(os.path.join(out_dir, f"r{rank}.npz"), labels=labels, conf=conf, acc=acc)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["copies", "parts"])
def test_two_rank_sharding_matches_single_process(mode, tmp_path):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), mode, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    prm = O.init_model(7)
    g1 = O.encode(O.gen_csa(8))
    if mode == "copies":
        g = O.batch(g1, 5)
        ref_pred, ref_conf, ref_acc, _ = O.predict_full(g, prm)
    else:
        g = O.batch(g1, 2)
        parts = O.regrow(g, O.topo_chunks(g.n, 5), 5)
        ref_pred, ref_conf, ref_acc = O.predict(g, parts, prm)
    for r in range(world):
        d = np.load(tmp_path / f"r{r}.npz")
        np.testing.assert_array_equal(d["labels"], ref_pred)
        np.testing.assert_array_equal(d["conf"], ref_conf)
        assert float(d["acc"]) == pytest.approx(ref_acc, abs=0)


def test_shard_ranges():
    n1 = 457
    got = [shard.copy_shard(r, 3, 16, n1) for r in range(3)]
    assert [s.count for s in got] == [5, 5, 6]
    assert sum(s.nodes for s in got) == 16 * n1
    assert [s.node_offset for s in got] == [0, 5 * n1, 10 * n1]
    assert shard.owned_parts(7, 1, 3) == [1, 4]
    with pytest.raises(ValueError):
        shard.copy_shard(0, 4, 2, n1)


# ---------------------------------------------------------------------------
# exact-halo mode X
# ---------------------------------------------------------------------------
def np_layer_fn(hg, prm, depth=4, in_dim=4, hidden=32, classes=5):
    """fp64 numpy restatement of one run_forward layer (src/gnn.cpp:37-52) on a
    local graph: m = D^-1 A h, h' = relu(h Ws + m Wn + b); last: h W_out + b_out."""
    import torch
    rp = hg.row_ptr.astype(np.int64)
    deg = np.diff(rp)
    rows = np.repeat(np.arange(hg.n), deg)
    offs = []
    off, fin = 0, in_dim
    for _ in range(depth):
        offs.append((off, fin))
        off += 2 * fin * hidden + hidden
        fin = hidden

    def layer(l, h):
        x = hg.features.astype(np.float64) if l == 0 else h.numpy()
        m = np.zeros_like(x)
        np.add.at(m, rows, x[hg.col_idx.astype(np.int64)])
        m = np.where(deg[:, None] > 0, m / np.maximum(deg, 1)[:, None], 0.0)
        o, fi = offs[l]
        ws = prm[o:o + fi * hidden].reshape(fi, hidden)
        wn = prm[o + fi * hidden:o + 2 * fi * hidden].reshape(fi, hidden)
        b = prm[o + 2 * fi * hidden:o + 2 * fi * hidden + hidden]
        z = np.maximum((x @ ws + m @ wn) + b, 0.0)
        if l + 1 == depth:
            wo = prm[off:off + hidden * classes].reshape(hidden, classes)
            bo = prm[off + hidden * classes:off + hidden * classes + classes]
            z = z @ wo + bo
        return torch.from_numpy(np.ascontiguousarray(z))
    return layer


def _xworker(rank, world, port, out_dir, partitioner="topo"):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        prm = O.init_model(7)
        g = O.encode(O.gen_csa(16))  # one copy: the parts straddle the circuit
        if partitioner == "topo":
            part_of = O.topo_chunks(g.n, world)
        else:  # the partition_multilevel replacement's cut
            part_of = O.partition_lp(g.row_ptr, g.col_idx, g.n, world)
        parts = O.regrow(g, part_of, world)
        plans = shard.halo_plans(part_of, [p.core_nodes for p in parts], [p.boundary_nodes for p in parts])
        local = O.materialize(g, parts[rank])
        ex = shard.HaloExchanger(plans[rank], 32, "cpu", torch.float64)  # index lists built once
        logits = shard.predict_exact(plans[rank], 4, np_layer_fn(local, prm), exchange=ex)
        np.savez(os.path.join(out_dir, f"x{rank}.npz"), core=parts[rank].core_nodes, logits=logits.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("partitioner", ["topo", "lp"])
def test_exact_halo_mode_matches_whole_graph(tmp_path, partitioner):
    """Mode X over 3 gloo ranks (parts straddling one 16-bit CSA copy; topo chunks
    or the LP partitioner's cut): the core rows' logits equal the whole-graph
    forward (predict_full semantics), which the reference's partitioned predict
    (mode R) does not reproduce."""
    world = 3
    mp.spawn(_xworker, args=(world, _free_port(), str(tmp_path), partitioner), nprocs=world, join=True)
    g = O.encode(O.gen_csa(16))
    prm = O.init_model(7)
    ref = O.forward(g, prm)
    got = np.zeros_like(ref)
    seen = np.zeros(g.n, bool)
    for r in range(world):
        d = np.load(os.path.join(tmp_path, f"x{r}.npz"))
        got[d["core"]] = d["logits"]
        seen[d["core"]] = True
    assert seen.all()
    np.testing.assert_allclose(got, ref, rtol=1e-9, atol=1e-12)
    # mode R on the same parts differs near the cuts (reference semantics)
    parts = O.regrow(g, O.topo_chunks(g.n, world), world)
    r_pred = np.zeros(g.n, np.float64)
    diff = 0.0
    for p in parts:
        lg = O.forward(O.materialize(g, p), prm)[: p.num_core]
        diff = max(diff, float(np.abs(lg - ref[p.core_nodes]).max()))
    assert diff > 1e-6


def test_halo_plans_consistent():
    g = O.encode(O.gen_csa(8))
    k = 4
    part_of = O.topo_chunks(g.n, k)
    parts = O.regrow(g, part_of, k)
    plans = shard.halo_plans(part_of, [p.core_nodes for p in parts], [p.boundary_nodes for p in parts])
    for r, pl in enumerate(plans):
        assert pl.num_local == parts[r].num_core + parts[r].boundary_nodes.shape[0]
        got = np.concatenate(pl.recv)
        assert np.array_equal(np.sort(got), np.arange(pl.num_core, pl.num_local))
        for q in range(k):
            sent_globals = parts[r].core_nodes[pl.send[q]]
            recv_globals = parts[q].local_to_global[plans[q].recv[r]]
            assert np.array_equal(sent_globals, recv_globals)
