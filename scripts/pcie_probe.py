import torch, time
n = 256 << 20
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
for _ in range(3):
    h.copy_(d, non_blocking=True); torch.cuda.synchronize()
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
s.record(); 
for _ in range(5): h.copy_(d, non_blocking=True)
e.record(); torch.cuda.synchronize(); print("D2H GB/s", 5 * n / s.elapsed_time(e) / 1e6)
s.record()
for _ in range(5): d.copy_(h, non_blocking=True)
e.record(); torch.cuda.synchronize(); print("H2D GB/s", 5 * n / s.elapsed_time(e) / 1e6)
# chunked D2H 8 x 32MB
s.record()
for i in range(8): h[i*(n//8):(i+1)*(n//8)].copy_(d[i*(n//8):(i+1)*(n//8)], non_blocking=True)
e.record(); torch.cuda.synchronize(); print("D2H chunked GB/s", n / s.elapsed_time(e) / 1e6)
