"""Host-side cost of one application (enqueue only, no sync): Python API vs direct C ABI."""
import os, sys, time
import ctypes as C
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_08427_b200 as rq  # noqa: E402
from paper_1708_08427_b200 import _lib as L  # noqa: E402
from paper_1708_08427_b200.workloads import make_config  # noqa: E402

pos, off = make_config(2, seed=1000, scale=0.05)
N, m = int(off[-1]), len(off) - 1
op = rq.MultiBodyOperator(rq.MultiBodyModel.from_arrays(pos, off))
v = torch.randn(3 * N, dtype=torch.float64, device="cuda")
out = torch.empty(3 * N - 6 * m, dtype=torch.float64, device="cuda")
lib, h = L.lib(), op.plan.handle
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for name, f in (("python op.apply", lambda: op.apply("qtilde_v", v)),
                ("C rq_apply_ex", lambda: lib.rq_apply_ex(h, L.OP_QTILDE_V, v.data_ptr(), out.data_ptr(), 1, st, 7))):
    for _ in range(20): f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200): f()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{name:18s} host {1e6 * (t1 - t0) / 200:7.1f} us/apply   (device-bound total {1e6 * (t2 - t0) / 200:7.1f} us)")
