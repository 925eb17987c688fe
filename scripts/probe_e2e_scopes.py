"""Per-scope GPU time (library event profiler) inside groot_classify_aig on the
1024-bit CSA b16 e2e workload, against the call's wall time: where the e2e
call's time goes beyond the device-resident forward.
usage: python scripts/probe_e2e_scopes.py [reps]"""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_18297_b200 import api  # noqa: E402
from paper_2511_18297_b200._lib import check, lib  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
L = lib()
c = api.gen_csa_multiplier(1024)
model = api.load_model(os.path.join(ROOT, "tests", "golden", "trained_csa8.asg1"))
ands = torch.from_numpy(np.ascontiguousarray(c.aig.and_lits)).pin_memory()
outs = torch.from_numpy(np.ascontiguousarray(c.aig.out_lits)).pin_memory()
lab = torch.from_numpy(np.ascontiguousarray(c.labels)).pin_memory()
pred = torch.empty(16 * c.labels.shape[0], dtype=torch.uint8).pin_memory()
conf = (C.c_uint64 * 25)()
acc = C.c_double()


def call():
    check(L.groot_classify_aig(model.handle, c.aig.num_inputs, c.aig.num_ands, C.c_void_p(ands.data_ptr()),
                               int(outs.numel()), C.c_void_p(outs.data_ptr()), C.c_void_p(lab.data_ptr()), 16,
                               C.c_void_p(pred.data_ptr()), conf, C.byref(acc)))


for _ in range(2):
    call()
L.groot_profile_enable(1)
t0 = time.perf_counter()
for _ in range(reps):
    call()
wall = (time.perf_counter() - t0) / reps * 1e3
maxk = 32
names = C.create_string_buffer(48 * maxk)
tot = (C.c_double * maxk)()
cnt = (C.c_uint64 * maxk)()
nk = C.c_uint32()
check(L.groot_profile_read(maxk, names, tot, cnt, C.byref(nk)))
L.groot_profile_enable(0)
s = 0.0
for i in range(min(nk.value, maxk)):
    nm = names.raw[48 * i:48 * (i + 1)].split(b"\0")[0].decode()
    s += tot[i] / reps
    print(f"{nm:24s} {tot[i] / reps:8.3f} ms/call  launches/call {cnt[i] / reps:.1f}")
print(f"scopes {s:.2f} ms of {wall:.2f} ms wall per call")
