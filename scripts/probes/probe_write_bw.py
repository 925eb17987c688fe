import torch, time
x = torch.empty(int(17.16e9)//4, dtype=torch.float32, device="cuda")
y = torch.empty(int(3.4e9)//4, dtype=torch.float32, device="cuda")
for _ in range(3): x.zero_()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): x.zero_()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)/5
print(f"write-only 17.16 GB: {ms:.3f} ms = {17.16/ms:.2f} TB/s")
z = torch.empty(int(3.4e9)//4, dtype=torch.float32, device="cuda")
e0.record()
for _ in range(5): z.copy_(y)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)/5
print(f"copy 3.4 GB: {ms:.3f} ms = {6.8/ms:.2f} TB/s (r+w)")
