"""Host link and host memory probe: pinned H2D / D2H / both at once (98 MB, config-2 vector
size), and multi-threaded memcpy pageable -> pinned (the staging step of the numpy path)."""
import ctypes
import os
import threading
import time

import torch

NB = 98_304_000
dev = torch.empty(NB // 8, dtype=torch.float64, device="cuda")
dev2 = torch.empty(NB // 8, dtype=torch.float64, device="cuda")
ph = torch.empty(NB // 8, dtype=torch.float64, pin_memory=True)
ph2 = torch.empty(NB // 8, dtype=torch.float64, pin_memory=True)
pg = torch.randn(NB // 8, dtype=torch.float64)  # pageable
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


def h2d():
    with torch.cuda.stream(s1):
        dev.copy_(ph, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        ph2.copy_(dev2, non_blocking=True)


def both():
    h2d()
    d2h()


for name, fn, nbytes in (("H2D", h2d, NB), ("D2H", d2h, NB), ("H2D+D2H", both, 2 * NB)):
    t = timed(fn)
    print(f"{name:8s} {t * 1e3:7.3f} ms  {nbytes / t / 1e9:6.1f} GB/s")

libc = ctypes.CDLL("libc.so.6")
libc.memcpy.restype = ctypes.c_void_p
libc.memcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t]
src, dst = pg.data_ptr(), ph.data_ptr()
for T in (1, 4, 8, 16, 32):
    if T > (os.cpu_count() or 1):
        break
    piece = 4 << 20
    n = (NB + piece - 1) // piece

    def run():
        def w(t):
            for i in range(t, n, T):
                off = i * piece
                libc.memcpy(dst + off, src + off, min(piece, NB - off))
        th = [threading.Thread(target=w, args=(t,)) for t in range(T)]
        for x in th:
            x.start()
        for x in th:
            x.join()

    t = timed(run, 5)
    print(f"memcpy pageable->pinned {T:2d} threads {t * 1e3:7.3f} ms  {NB / t / 1e9:6.1f} GB/s")
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
