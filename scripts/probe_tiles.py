"""Per-tile time of the fused layer vs graph size (L2-resident vs HBM-resident features)."""
import os, sys, ctypes as C
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_18297_b200 import api
from paper_2511_18297_b200._lib import lib, check
L = lib()
api.set_stream(torch.cuda.current_stream().cuda_stream)
model = api.init_model(7)
for w, b in [(128, 2), (128, 4), (256, 2), (256, 8), (512, 16), (1024, 16)]:
    c = api.gen_csa_multiplier(w); g = api.batch(api.encode(c.aig, c.labels), b)
    n = g.n
    cls = torch.empty(n, dtype=torch.uint8, device="cuda")
    for i in range(2):
        check(L.groot_predict_full_dev(model.handle, g.handle, C.c_void_p(cls.data_ptr()), None, None))
    L.groot_profile_enable(1)
    for i in range(5):
        check(L.groot_predict_full_dev(model.handle, g.handle, C.c_void_p(cls.data_ptr()), None, None))
    names = C.create_string_buffer(48 * 16); tot = (C.c_double * 16)(); cnt = (C.c_uint64 * 16)(); nk = C.c_uint32()
    check(L.groot_profile_read(16, names, tot, cnt, C.byref(nk)))
    L.groot_profile_enable(0)
    k = {names.raw[48*i:48*(i+1)].split(b"\0")[0].decode(): tot[i]/cnt[i] for i in range(nk.value)}
    tiles = (n + 127) // 128
    ms = k["sage_layer_tc"]
    print(f"w={w} b={b} n={n} H={n*128/1e6:.0f}MB tc={ms:.3f}ms per-tile/SM={ms*1e3/(tiles/148):.2f}us  L0={k['sage_layer0']:.3f}")
    del g, cls
