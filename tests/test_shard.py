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
