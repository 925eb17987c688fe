"""Quick device timing of the forward on a CSA graph (development probe, not the bench)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2511_18297_b200 import api

width = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
copies = int(sys.argv[2]) if len(sys.argv) > 2 else 16
t0 = time.time()
c = api.gen_csa_multiplier(width)
t1 = time.time()
g1 = api.encode(c.aig, c.labels)
g = api.batch(g1, copies) if copies > 1 else g1
torch.cuda.synchronize()
t2 = time.time()
n, nnz, E = g.n, g.nnz, g.num_undirected_edges()
print(f"gen {t1-t0:.2f}s encode+batch {t2-t1:.2f}s n={n} nnz={nnz} E={E}", flush=True)
model = api.init_model(7)
s = torch.cuda.current_stream()
api.set_stream(s.cuda_stream)
cls = torch.empty(n, dtype=torch.uint8, device="cuda")
from paper_2511_18297_b200._lib import lib, check
for i in range(3):
    check(lib().groot_predict_full_dev(model.handle, g.handle, cls.data_ptr(), None, None))
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
K = 10
ev[0].record()
for i in range(K):
    check(lib().groot_predict_full_dev(model.handle, g.handle, cls.data_ptr(), None, None))
ev[1].record()
torch.cuda.synchronize()
ms = ev[0].elapsed_time(ev[1]) / K
print(f"forward+classify {ms:.3f} ms/step  -> {E/ms*1e3/1e9:.3f} G edges/s; roofline frac {114386760032*(E/268107776)/ (ms*1e-3) / 6549.4e9:.3f}")
# standalone spmm f=32
dense = torch.randn(n, 32, device="cuda")
out = torch.empty_like(dense)
for i in range(2):
    check(lib().groot_spmm_mean_dev(g.handle, dense.data_ptr(), 32, out.data_ptr()))
ev[0].record()
for i in range(K):
    check(lib().groot_spmm_mean_dev(g.handle, dense.data_ptr(), 32, out.data_ptr()))
ev[1].record(); torch.cuda.synchronize()
ms2 = ev[0].elapsed_time(ev[1]) / K
B = 4*(n+1) + 4*nnz + 2*4*32*n
print(f"spmm_mean f=32 {ms2:.3f} ms -> {B/ms2/1e6:.1f} GB/s ({B/ms2/1e6/6549.4:.3f} of 6549.4)")
