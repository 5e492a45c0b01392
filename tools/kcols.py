"""Device time of Q~v for (rows, k) blocks on config 2 (k columns), single-RHS column loop vs multi-RHS kernels."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_1708_08427_b200 as rq  # noqa: E402
from paper_1708_08427_b200.workloads import make_config  # noqa: E402

pos, off = make_config(2, seed=1000, scale=0.25)
N, m = int(off[-1]), len(off) - 1
op = rq.MultiBodyOperator(rq.MultiBodyModel.from_arrays(pos, off))
for k in (1, 2, 3, 4, 6, 8, 16):
    v = torch.randn(3 * N, k, dtype=torch.float64, device="cuda")
    for _ in range(3):
        op.apply("qtilde_v", v)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        op.apply("qtilde_v", v)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"min={os.environ.get('RQ_MRHS_MIN', '8')} k={k:3d}: {ms:.3f} ms  {N * k / ms / 1e6:.2f} G bead-RHS/s", flush=True)
