"""Time the host-buffer C-ABI path (rq_apply_host) on config 2 for several segment settings."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_08427_b200 as rq  # noqa: E402
from paper_1708_08427_b200 import _lib as L  # noqa: E402
from paper_1708_08427_b200.workloads import make_config  # noqa: E402

pos, off = make_config(2, seed=1000, scale=float(sys.argv[1]) if len(sys.argv) > 1 else 1.0)
N, m = int(off[-1]), len(off) - 1
op = rq.MultiBodyOperator(rq.MultiBodyModel.from_arrays(pos, off))
h = op.plan.handle
lib = L.lib()
hv = torch.randn(3 * N, dtype=torch.float64).pin_memory()
hg = torch.randn(3 * N - 6 * m, dtype=torch.float64).pin_memory()
o1 = torch.empty(3 * N - 6 * m, dtype=torch.float64).pin_memory()
o2 = torch.empty(3 * N, dtype=torch.float64).pin_memory()
for segs, mb in [(4, 2), (6, 2), (8, 2), (10, 2), (12, 1)]:
    os.environ["RQ_HOST_SEGS"] = str(segs)
    os.environ["RQ_HOST_SEG_MB"] = str(mb)
    for _ in range(2):
        L.check(lib.rq_apply_host(h, L.OP_QTILDE_V, hv.data_ptr(), o1.data_ptr(), 1))
        L.check(lib.rq_apply_host(h, L.OP_QTILDE_TV, hg.data_ptr(), o2.data_ptr(), 1))
    t0 = time.perf_counter()
    n = 10
    for _ in range(n):
        L.check(lib.rq_apply_host(h, L.OP_QTILDE_V, hv.data_ptr(), o1.data_ptr(), 1))
        L.check(lib.rq_apply_host(h, L.OP_QTILDE_TV, hg.data_ptr(), o2.data_ptr(), 1))
    dt = (time.perf_counter() - t0) / n
    print(f"segs {segs:4d} mb {mb}: {dt*1e3:7.3f} ms/step  {N/dt/1e9:6.3f} G beads/s", flush=True)
# raw copy speeds
d = torch.empty(3 * N, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    d.copy_(hv[:3 * N - 6 * m].new_empty(0) if False else hv, non_blocking=True)
torch.cuda.synchronize()
print(f"H2D {10 * hv.numel() * 8 / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
t0 = time.perf_counter()
for _ in range(10):
    o2.copy_(d, non_blocking=True)
torch.cuda.synchronize()
print(f"D2H {10 * o2.numel() * 8 / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
