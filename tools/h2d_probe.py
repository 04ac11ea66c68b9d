"""Pinned H2D rate: one 134 MB copy vs two concurrent copies on two streams (debug tool)."""
import time
import torch

n = 4096 * 4096
a = torch.empty(n, dtype=torch.float64).pin_memory()
b = torch.empty(n, dtype=torch.float64).pin_memory()
da = torch.empty(n, dtype=torch.float64, device="cuda")
db = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(3):
    da.copy_(a, non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    da.copy_(a, non_blocking=True)
    db.copy_(b, non_blocking=True)
torch.cuda.synchronize()
seq = (time.perf_counter() - t0) / 10
t0 = time.perf_counter()
for _ in range(10):
    with torch.cuda.stream(s1):
        da.copy_(a, non_blocking=True)
    with torch.cuda.stream(s2):
        db.copy_(b, non_blocking=True)
    torch.cuda.synchronize()
par = (time.perf_counter() - t0) / 10
print(f"2 x 134 MB: sequential {seq * 1e3:.2f} ms ({2 * n * 8 / seq / 1e9:.1f} GB/s), "
      f"two streams {par * 1e3:.2f} ms ({2 * n * 8 / par / 1e9:.1f} GB/s)")
