#!/usr/bin/env python
"""bench.py — GNN inference edges/s on the 1024-bit CSA multiplier AIG, batch 16.

Contract (see task statement / DESIGN.md "Measurement"):
  python bench.py --gpus N --steps K --warmup W        (N>1 via torch.distributed.run)
  python bench.py --impl reference ...                  (the reference CPU path)
One JSON line on rank 0.

A *step* is one pass of the hot path over the resident batch: layer forward of
the 4-layer GraphSAGE + classify (argmax + confusion) over every node of
batch(encode(gen_csa_multiplier(1024)), 16) — 134,103,056 nodes, 268,107,776
edges per GPU (weak scaling: every rank owns 16 copies; global batch 16*N).
``value`` = edges (undirected fwd_edges, all ranks) / max-over-ranks device
time. ``e2e`` = the same metric through the public C ABI call
groot_classify_aig with the AIG in pinned host memory: H2D of the AIG literals
+ labels, device encode -> batch -> forward -> classify, D2H of the classes.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GNN inference edges/s, 1024-bit CSA bs16; SpMM HBM GB/s vs roofline"
UNIT = "edges/s"
MODEL_FILE = os.path.join(ROOT, "tests", "golden", "trained_csa8.asg1")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--width", type=int, default=1024)
    p.add_argument("--circuit", choices=["csa", "booth"], default="csa",
                   help="multiplier family (booth = BASELINE config 3's radix-4 Booth AIG)")
    p.add_argument("--batch", type=int, default=16, help="copies per GPU")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=None)
    return p.parse_args()


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 50 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            return self
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        return self.summary()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# reference CPU path (oracle/_ref = the reference's own compiled sources)
# ---------------------------------------------------------------------------
class RefSample:
    """Bounded sample of the workload on the reference CPU path: `count` consecutive
    topo partitions (regrown, k parts) from the middle of one 1024-bit copy,
    predicted with the reference's partition-parallel predict (default_pool =
    all host threads). Edges counted = fwd_edges whose head node lies in the sample."""

    def __init__(self, width: int, circuit: str = "csa"):
        from oracle import pyoracle as O
        from oracle import pyref as R
        self.R = R
        self.kind = "reference"
        if not R.available():
            raise RuntimeError("oracle/_ref not built")
        self.workers = R.default_workers()
        self.k = 64
        while self.k < 4 * self.workers:
            self.k *= 2
        self.first = self.k // 8
        self.count = self.workers
        if circuit == "booth":  # the reference's own Aig + encode on our Booth AIG (no reference generator)
            from paper_2511_18297_b200 import api
            c = api.gen_booth_multiplier(width)
            _, self.g = R.aig_from_lits(c.aig.num_inputs, c.aig.and_lits, c.aig.out_lits)
        else:
            _, self.g = R.gen_csa(width)
        part = R.topo_chunks(self.g, self.k)
        self.parts = R.RefParts(self.g, part, self.k, True)
        edges = self.g.to_host().fwd_edges
        hp = part[edges[:, 1]]
        self.edges = int(((hp >= self.first) & (hp < self.first + self.count)).sum())
        self.params = O.load_model(MODEL_FILE)[0]
        self.desc = (f"{self.count} consecutive regrown topo parts (k={self.k}, parts {self.first}.."
                     f"{self.first + self.count - 1}) of one {width}-bit {circuit.upper()} copy = {self.edges} edges; "
                     f"reference predict (src/gnn.cpp:280) with aggregation by the compiled spmm::execute, "
                     f"dense h*W restated (Eigen absent)")

    def step(self):
        t = time.perf_counter()
        self.R.predict_parts(self.parts, self.first, self.count, self.params)
        return time.perf_counter() - t


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    try:
        s = RefSample(args.width, args.circuit)
    except Exception as e:  # pragma: no cover
        print(json.dumps({"impl": "reference", "unavailable": f"reference CPU path not loadable: {e}"}))
        return
    for _ in range(args.warmup):
        s.step()
    times = [s.step() for _ in range(args.steps)]
    total = sum(times)
    value = s.edges * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (deterministic {args.circuit.upper()} generator)",
        "config": {"workload": f"{args.width}-bit {args.circuit.upper()} multiplier AIG, batch {args.batch} per GPU (sampled)",
                   "width": args.width, "batch": args.batch, "parallelism": "host threads"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": s.workers, "kind": s.kind, "sample": s.desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2511_18297_b200 import api
    from paper_2511_18297_b200._lib import check, lib
    import ctypes as C

    stream = torch.cuda.current_stream()
    api.set_stream(stream.cuda_stream)
    L = lib()

    # ---- setup (untimed): AIG on host, encode + batch on device ----
    circ = (api.gen_booth_multiplier if args.circuit == "booth" else api.gen_csa_multiplier)(args.width)
    g1 = api.encode(circ.aig, circ.labels)
    g = api.batch(g1, args.batch) if args.batch > 1 else g1
    n, nnz, E = g.n, g.nnz, g.num_undirected_edges()
    model = api.load_model(MODEL_FILE)
    cls = torch.empty(n, dtype=torch.uint8, device="cuda")
    conf = torch.zeros(25, dtype=torch.int64, device="cuda")

    def step():
        check(L.groot_predict_full_dev(model.handle, g.handle, C.c_void_p(cls.data_ptr()), None,
                                       C.c_void_p(conf.data_ptr())))
        if world > 1:  # global confusion / accuracy: the only exchange of the path
            dist.all_reduce(conf)

    for _ in range(max(args.warmup, 3)):
        conf.zero_()
        step()
    torch.cuda.synchronize()

    # ---- timed region: device-resident steps ----
    sampler = ClockSampler(local).start()
    time.sleep(0.3)
    L.groot_profile_enable(1)
    launches0 = L.groot_kernel_launches()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = L.groot_kernel_launches() - launches0
    clocks = sampler.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # per-kernel event totals over the timed region (recorded on the launching stream)
    maxk = 32
    names = C.create_string_buffer(48 * maxk)
    tot = (C.c_double * maxk)()
    cnt = (C.c_uint64 * maxk)()
    nk = C.c_uint32()
    check(L.groot_profile_read(maxk, names, tot, cnt, C.byref(nk)))
    L.groot_profile_enable(0)
    kernels = {}
    for i in range(min(nk.value, maxk)):
        nm = names.raw[48 * i:48 * (i + 1)].split(b"\0")[0].decode()
        kernels[nm] = {"ms_per_launch": tot[i] / max(cnt[i], 1), "launches": int(cnt[i]),
                       "ms_per_step": tot[i] / args.steps}

    # the same forward with layer 0 materialized (GROOT_L0_KEYED=0: n x 128 B layer-0 rows
    # written and read back), reported beside the keyed default for transparency
    os.environ["GROOT_L0_KEYED"] = "0"
    for _ in range(2):
        step()
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    del os.environ["GROOT_L0_KEYED"]
    ms_mat = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms_mat], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_mat = float(t.item())

    # row classifier output (HD band) for the algorithmic-byte accounting
    deg = None
    num_hd = 0
    hd_nnz = 0
    try:
        rp = g.row_ptr
        deg = np.diff(rp)
        thr = int(os.environ.get("GROOT_HD_THRESHOLD", "128"))
        num_hd = int((deg >= thr).sum())
        hd_nnz = int(deg[deg >= thr].sum())
        del rp
    except Exception:
        pass

    peak, peak_src = measured_peaks()
    # dominant kernel: the fused 32->32 layer (gather + tcgen05 transform + epilogue)
    ld_nnz = nnz - hd_nnz
    bytes_tc = 4 * (n + 1) + 4 * ld_nnz + 128 * n + 128 * n + 128 * num_hd
    k_tc = kernels.get("sage_layer_tc")
    roof = None
    if k_tc:
        achieved = bytes_tc / (k_tc["ms_per_launch"] * 1e-3) / 1e9
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
                summ = json.load(f)
                traffic = summ.get("kernels", {}).get("sage_layer_tc", {}).get("dram_bytes_per_launch")
        except Exception:
            pass
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": "sage_tile_kernel<kModeLayer> (tile-planned fused 32->32 SAGE layer)",
                "algorithmic_bytes_per_launch": bytes_tc, "peak_source": peak_src}
    # whole forward: CSR / plan structure, layer inputs and outputs, u8 classes.
    # Keyed layer 0 (records -> u8 entry ids) replaces the n x 128 B layer-0 rows written by
    # layer 0 and read back by layer 1 with one byte per row each way.
    keyed = "l0_keys" in kernels
    depth = 4
    csr, ld = 4 * (n + 1) + 4 * nnz, 4 * (n + 1) + 4 * ld_nnz
    l0 = csr + 4 * n + (n if keyed else 128 * n)
    l1 = ld + (n if keyed else 128 * n) + 128 * n + 128 * num_hd
    mid = ld + 128 * n + 128 * n + 128 * num_hd
    last = ld + 128 * n + n + 128 * num_hd
    full_bytes = l0 + l1 + mid * (depth - 3) + last + 2 * n
    k_x = kernels.get("sage_layer1_xform")
    l1_roof = None
    if k_x:  # keyed transform-first layer 1 (a gather-sum: no input rows, table in shared memory)
        ach = l1 / (k_x["ms_per_launch"] * 1e-3) / 1e9
        l1_roof = {"kernel": "sage_tile_kernel<kModeXform, true> (keyed transform-first layer 1)", "bound": "hbm",
                   "algorithmic_bytes_per_launch": l1, "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak}

    # standalone SpMM (mean aggregation, f=32): the metric's "SpMM HBM GB/s"
    dense = torch.randn(n, 32, device="cuda")
    outm = torch.empty_like(dense)
    for _ in range(2):
        check(L.groot_spmm_mean_dev(g.handle, C.c_void_p(dense.data_ptr()), 32, C.c_void_p(outm.data_ptr())))
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(args.steps):
        check(L.groot_spmm_mean_dev(g.handle, C.c_void_p(dense.data_ptr()), 32, C.c_void_p(outm.data_ptr())))
    ev1.record(stream)
    torch.cuda.synchronize()
    spmm_ms = ev0.elapsed_time(ev1) / args.steps
    spmm_bytes = 4 * (n + 1) + 4 * nnz + 2 * 128 * n
    spmm = {"ms": spmm_ms, "algorithmic_bytes": spmm_bytes, "achieved_gbs": spmm_bytes / spmm_ms / 1e6,
            "frac": spmm_bytes / spmm_ms / 1e6 / peak}
    del dense, outm

    # ---- e2e through the public C ABI with pinned host buffers ----
    del g
    torch.cuda.synchronize()
    ands_h = torch.from_numpy(circ.aig.and_lits.view(np.int32).reshape(-1)).pin_memory()
    outs_h = torch.from_numpy(circ.aig.out_lits.view(np.int32)).pin_memory()
    lab_h = torch.from_numpy(circ.labels).pin_memory()
    pred_h = torch.empty(n, dtype=torch.uint8).pin_memory()
    conf_h = (C.c_uint64 * 25)()
    acc = C.c_double()

    def e2e_call():
        check(L.groot_classify_aig(model.handle, circ.aig.num_inputs, circ.aig.num_ands,
                                   C.c_void_p(ands_h.data_ptr()), int(outs_h.numel()),
                                   C.c_void_p(outs_h.data_ptr()), C.c_void_p(lab_h.data_ptr()), args.batch,
                                   C.c_void_p(pred_h.data_ptr()), conf_h, C.byref(acc)))

    e2e_steps = args.e2e_steps or max(3, min(args.steps, 10))
    for _ in range(2):
        e2e_call()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_call()
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    h2d = ands_h.numel() * 4 + outs_h.numel() * 4 + lab_h.numel()
    d2h = pred_h.numel() + 25 * 8
    accuracy = acc.value

    # ---- CPU baseline (rank 0, N=1 only) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            s = RefSample(args.width, args.circuit)
            s.step()
            reps = 4
            tt = sum(s.step() for _ in range(reps))
            cpu = {"value": s.edges * reps / tt, "unit": UNIT, "cores": s.workers, "kind": s.kind,
                   "sample": s.desc}
        except Exception as e:
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        value = E * world / (ms * 1e-3)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32 (3xTF32 tcgen05 transform, fp32 accumulate)",
            "data": f"synthetic (deterministic {args.circuit.upper()} multiplier generator; trained 8-bit ASG1 weights)",
            "config": {"workload": f"{args.width}-bit {args.circuit.upper()} multiplier AIG, batch {args.batch} per GPU "
                                   f"(4-layer GraphSAGE 4-32-32-32-32 + 32->5 head, predict_full)",
                       "width": args.width, "batch_per_gpu": args.batch, "global_batch": args.batch * world,
                       "nodes_per_gpu": n, "edges_per_gpu": E, "nnz_per_gpu": nnz,
                       "parallelism": f"dp{world} (whole batch copies per GPU)" if world > 1 else "single GPU",
                       "l2": "inputs (>40 GB resident) far exceed L2; no flush"},
            "roofline": roof,
            "layer1_roofline": l1_roof,
            "materialized_layer0": {"ms_per_step": ms_mat, "value": E * world / (ms_mat * 1e-3), "unit": UNIT,
                                    "note": "same forward with GROOT_L0_KEYED=0 (layer-0 rows materialized)"},
            "forward_roofline": ({"algorithmic_bytes": full_bytes, "achieved_gbs": full_bytes / ms / 1e6,
                                  "frac": full_bytes / ms / 1e6 / peak, "keyed_layer0": keyed} if full_bytes else None),
            "spmm": spmm,
            "kernels": kernels,
            "cpu_baseline": cpu,
            "e2e": {"value": E * world / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s * 1e3,
                    "path": "groot_classify_aig (pinned host AIG -> encode -> batch -> predict_full -> host classes)"},
            "accuracy": accuracy,
            "clocks": clocks,
            "gpu_launches": int(launches),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
        rank, world, _ = dist_env()
        return
    run_ours(args)


if __name__ == "__main__":
    main()
