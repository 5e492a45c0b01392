"""One Q~v and one Q~^T g on config 2 (device-resident), for ncu captures of k_wave."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1708_08427_b200 as rq  # noqa: E402
from paper_1708_08427_b200.workloads import make_config  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
pos, off = make_config(cfg, seed=1000)
N, m = int(off[-1]), len(off) - 1
op = rq.MultiBodyOperator(rq.MultiBodyModel.from_arrays(pos, off))
v = torch.randn(3 * N, dtype=torch.float64, device="cuda")
g = torch.randn(3 * N - 6 * m, dtype=torch.float64, device="cuda")
op.apply("qtilde_v", v)
op.apply("qtilde_tv", g)
torch.cuda.synchronize()
