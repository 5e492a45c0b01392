"""Launch only the top-tree phase of Q~v / Q~^T v (for ncu), then time it.
argv: [reps] [bodies] [config]"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
import paper_1708_08427_b200 as rq  # noqa: E402
from paper_1708_08427_b200 import _lib as L  # noqa: E402
from paper_1708_08427_b200.workloads import make_config  # noqa: E402

cfg = int(sys.argv[3]) if len(sys.argv) > 3 else 2
pos, off = make_config(cfg, seed=1000)
mb = int(sys.argv[2]) if len(sys.argv) > 2 else len(off) - 1
off = off[: mb + 1]
pos = pos[: int(off[-1])]
N, m = int(off[-1]), len(off) - 1
op = rq.MultiBodyOperator(rq.MultiBodyModel.from_arrays(pos, off))
lib, h = L.lib(), op.plan.handle
s = torch.cuda.current_stream()
st = C.c_void_p(s.cuda_stream)
v = torch.randn(3 * N, dtype=torch.float64, device="cuda")
g = torch.randn(3 * N - 6 * m, dtype=torch.float64, device="cuda")
ov = torch.empty_like(g)
og = torch.empty_like(v)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for name, code, x, o in (("up", L.OP_QTILDE_V, v, ov), ("down", L.OP_QTILDE_TV, g, og)):
    for _ in range(3):
        L.check(lib.rq_apply_ex(h, code, x.data_ptr(), o.data_ptr(), 1, st, 3))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        L.check(lib.rq_apply_ex(h, code, x.data_ptr(), o.data_ptr(), 1, st, 2))
    b.record(s)
    torch.cuda.synchronize()
    print(f"cfg{cfg} m={mb} {name} top {a.elapsed_time(b) / reps * 1e3:.1f} us")
