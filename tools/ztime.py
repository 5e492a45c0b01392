"""Time Zf / Z^T u (device-resident CUDA tensors); argv: [config=2] [scale=1]."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1708_08427_b200 as rq  # noqa: E402
from paper_1708_08427_b200.workloads import make_config  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
pos, off = make_config(cfg, seed=1000, scale=float(sys.argv[2]) if len(sys.argv) > 2 else 1.0)
N, m = int(off[-1]), len(off) - 1
op = rq.MultiBodyOperator(rq.MultiBodyModel.from_arrays(pos, off))
f = torch.randn(3 * N, dtype=torch.float64, device="cuda")
u = torch.randn(6 * m, dtype=torch.float64, device="cuda")
for name, fn in (("zf", lambda: op.zf(f)), ("ztu", lambda: op.ztu(u))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 50
    print(f"{name}: {ms:.3f} ms  {N / ms / 1e6:.2f} G beads/s  {48 * N / ms / 1e6:.0f} GB/s (48 B/bead)")
