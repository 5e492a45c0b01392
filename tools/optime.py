"""Device time per application of each operator on config 2 (or argv[1]; inputs resident)."""
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
_i = op.plan.info()
print({k: _i[k] for k in ("n_streams", "n_steps", "node_slots", "stage_bytes", "sweep_smem", "sweep_ctas_per_sm", "sweep_bytes")})
for name, x in (("qtilde_v", v), ("qtilde_tv", g), ("both", None)):
    def run():
        if x is None:
            op.apply("qtilde_v", v)
            op.apply("qtilde_tv", g)
        else:
            op.apply(name, x)
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50 if cfg != 4 else 5):
        run()
    b.record()
    torch.cuda.synchronize()
    print(f"{name}: {a.elapsed_time(b) / (50 if cfg != 4 else 5):.4f} ms")
