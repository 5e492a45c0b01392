"""Q~V and Q~^T G on (rows, k) blocks (config 5 bodies, default 300 of them, k = 32),
device-resident, for ncu captures and A/B timing of k_mrhs.  argv: [bodies] [k] [reps]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1708_08427_b200 as rq  # noqa: E402
from paper_1708_08427_b200.workloads import ellipsoid_batch  # noqa: E402

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 300
k = int(sys.argv[2]) if len(sys.argv) > 2 else 32
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
pos, off = ellipsoid_batch([8192] * nb, seed=1000)
N, m = int(off[-1]), len(off) - 1
op = rq.MultiBodyOperator(rq.MultiBodyModel.from_arrays(pos, off))
V = torch.randn(3 * N, k, dtype=torch.float64, device="cuda")
G = torch.randn(3 * N - 6 * m, k, dtype=torch.float64, device="cuda")
op.apply("qtilde_v", V)
op.apply("qtilde_tv", G)
torch.cuda.synchronize()
if reps > 1:
    t = {}
    for name, x in (("qtilde_v", V), ("qtilde_tv", G)):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            op.apply(name, x)
        b.record()
        torch.cuda.synchronize()
        t[name] = a.elapsed_time(b) / reps
    print(f"bodies {nb} k {k}: qtilde_v {t['qtilde_v']:.4f} ms  qtilde_tv {t['qtilde_tv']:.4f} ms")
