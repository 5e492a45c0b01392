"""H2D and D2H bandwidth alone and concurrently (pinned host memory, separate streams)."""
import time

import torch

n = 98_304_000 // 8 * 4  # 4 x 98 MB
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d_a.copy_(h_in, non_blocking=True)
    h_out.copy_(d_b, non_blocking=True)
torch.cuda.synchronize()
for name, fn in (("h2d", lambda: d_a.copy_(h_in, non_blocking=True)), ("d2h", lambda: h_out.copy_(d_b, non_blocking=True))):
    t0 = time.perf_counter()
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    print(name, f"{5 * n * 8 / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
t0 = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
torch.cuda.synchronize()
el = time.perf_counter() - t0
print(f"concurrent: {5 * n * 8 / el / 1e9:.1f} GB/s each direction, {2 * 5 * n * 8 / el / 1e9:.1f} GB/s total")
