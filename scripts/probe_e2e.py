"""groot_classify_aig on the 1024-bit CSA b16 workload (e2e path) — a few calls, for
`ncu --metrics gpu__time_duration.sum` launch lists and host timing (GROOT_HOST_TIMING=1)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_18297_b200 import api  # noqa: E402
from paper_2511_18297_b200._lib import check, lib  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = api.gen_csa_multiplier(1024)
model = api.load_model(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                                    "trained_csa8.asg1"))
ands = torch.from_numpy(np.ascontiguousarray(c.aig.and_lits)).pin_memory()
outs = torch.from_numpy(np.ascontiguousarray(c.aig.out_lits)).pin_memory()
lab = torch.from_numpy(np.ascontiguousarray(c.labels)).pin_memory()
pred = torch.empty(16 * (c.labels.shape[0]), dtype=torch.uint8).pin_memory()
conf = (C.c_uint64 * 25)()
acc = C.c_double()
import time
for _ in range(reps):
    t0 = time.perf_counter()
    check(lib().groot_classify_aig(model.handle, c.aig.num_inputs, c.aig.num_ands, C.c_void_p(ands.data_ptr()),
                                   int(outs.numel()), C.c_void_p(outs.data_ptr()), C.c_void_p(lab.data_ptr()), 16,
                                   C.c_void_p(pred.data_ptr()), conf, C.byref(acc)))
    print(f"call {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
print("accuracy", acc.value)
