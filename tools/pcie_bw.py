"""Pinned host<->device copy bandwidth (the e2e ceiling), one direction and both at once."""
import torch
n = 1 << 28  # 1 GiB fp32
h = torch.empty(n, dtype=torch.float32).pin_memory()
h2 = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
d2 = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); d.copy_(h, non_blocking=True); e1.record(); torch.cuda.synchronize()
print(f"H2D {4 * n / e0.elapsed_time(e1) / 1e6:.1f} GB/s")
e0.record(); h.copy_(d, non_blocking=True); e1.record(); torch.cuda.synchronize()
print(f"D2H {4 * n / e0.elapsed_time(e1) / 1e6:.1f} GB/s")
torch.cuda.synchronize()
import time
t = time.perf_counter()
with torch.cuda.stream(s1):
    d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2):
    h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
print(f"duplex {2 * 4 * n / (time.perf_counter() - t) / 1e9:.1f} GB/s total")
