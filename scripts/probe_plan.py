"""Time the per-graph preprocessing of the device path on a CSA graph: encode,
batch, row classifier + tile plan (first forward minus steady forward)."""
import ctypes as C
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_18297_b200 import api  # noqa: E402
from paper_2511_18297_b200._lib import check, lib  # noqa: E402

w = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
b = int(sys.argv[2]) if len(sys.argv) > 2 else 16
api.set_stream(torch.cuda.current_stream().cuda_stream)
L = lib()
c = api.gen_csa_multiplier(w)
model = api.init_model(7)
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g1 = api.encode(c.aig, c.labels)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    g = api.batch(g1, b)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    cls = torch.empty(g.n, dtype=torch.uint8, device="cuda")
    L.groot_profile_enable(1)
    check(L.groot_predict_full_dev(model.handle, g.handle, C.c_void_p(cls.data_ptr()), None, None))
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    check(L.groot_predict_full_dev(model.handle, g.handle, C.c_void_p(cls.data_ptr()), None, None))
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    names = C.create_string_buffer(48 * 16)
    tot = (C.c_double * 16)()
    cnt = (C.c_uint64 * 16)()
    nk = C.c_uint32()
    check(L.groot_profile_read(16, names, tot, cnt, C.byref(nk)))
    L.groot_profile_enable(0)
    prof = {names.raw[48 * i:48 * (i + 1)].split(b"\0")[0].decode(): round(tot[i], 2) for i in range(nk.value)}
    print(f"rep {rep}: encode {1e3*(t1-t0):.1f} ms batch {1e3*(t2-t1):.1f} ms first forward {1e3*(t3-t2):.1f} ms "
          f"steady forward {1e3*(t4-t3):.1f} ms -> per-graph prep {1e3*(t3-t2-(t4-t3)):.1f} ms")
    print("  kernel totals (ms, both forwards):", prof)
    del g, g1
