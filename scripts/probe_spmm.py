"""Time the standalone mean-aggregation SpMM (f=32) on the 1024-bit b16 graph."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_18297_b200 import api
from paper_2511_18297_b200._lib import lib, check
import ctypes as C
w, b = int(sys.argv[1]), int(sys.argv[2])
c = api.gen_csa_multiplier(w); g = api.batch(api.encode(c.aig, c.labels), b)
n, nnz = g.n, g.nnz
api.set_stream(torch.cuda.current_stream().cuda_stream)
dense = torch.randn(n, 32, device="cuda"); out = torch.empty_like(dense)
L = lib()
L.groot_profile_enable(1)
for i in range(12):
    check(L.groot_spmm_mean_dev(g.handle, C.c_void_p(dense.data_ptr()), 32, C.c_void_p(out.data_ptr())))
torch.cuda.synchronize()
names = C.create_string_buffer(48 * 8); tot = (C.c_double * 8)(); cnt = (C.c_uint64 * 8)(); nk = C.c_uint32()
check(L.groot_profile_read(8, names, tot, cnt, C.byref(nk)))
res = {names.raw[48*i:48*(i+1)].split(b"\0")[0].decode(): tot[i] / cnt[i] for i in range(nk.value)}
B = 4 * (n + 1) + 4 * nnz + 2 * 128 * n
ms = res.get("spmm_mean32", 0)
print(f"occ={os.environ.get('GROOT_SPMM_BLOCKS')} {res} -> LD kernel {B/ms/1e6:.0f} GB/s (bytes incl. HD share)")
