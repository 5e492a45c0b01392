"""Cost of page-locking a user (pageable) numpy array in place with cudaHostRegister, vs staging
it through pinned memory: register / H2D / unregister times for a config-2 vector (98 MB)."""
import ctypes
import time

import numpy as np
import torch

cudart = ctypes.CDLL("libcudart.so") if False else None
rt = torch.cuda.cudart()
NB = 98_304_000
a = np.random.default_rng(0).normal(size=NB // 8)
dev = torch.empty(NB // 8, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
for flags, name in ((0, "default"), (8, "read-only")):
    ts = []
    for it in range(6):
        t0 = time.perf_counter()
        r = rt.cudaHostRegister(a.ctypes.data, NB, flags)
        t1 = time.perf_counter()
        dev.copy_(torch.from_numpy(a), non_blocking=True)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        rt.cudaHostUnregister(a.ctypes.data)
        t3 = time.perf_counter()
        ts.append((t1 - t0, t2 - t1, t3 - t2))
        if it == 0:
            print(name, "register rc", r)
    m = np.median(np.array(ts[1:]), axis=0) * 1e3
    print(f"{name}: register {m[0]:.3f} ms, H2D {m[1]:.3f} ms ({NB / m[1] / 1e6:.1f} GB/s), unregister {m[2]:.3f} ms")
# fresh (never touched) array: registration also faults the pages in
b = np.empty(NB // 8)
t0 = time.perf_counter()
rt.cudaHostRegister(b.ctypes.data, NB, 0)
t1 = time.perf_counter()
rt.cudaHostUnregister(b.ctypes.data)
print(f"untouched array: register {1e3 * (t1 - t0):.3f} ms")
