"""Fixed host overhead of rq_apply_host (tiny model) and its segment scaling on config 2."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_08427_b200 as rq  # noqa: E402
from paper_1708_08427_b200 import _lib as L  # noqa: E402
from paper_1708_08427_b200.workloads import make_config, ellipsoid_batch  # noqa: E402

lib = L.lib()
def timeit(h, N, m, reps=20):
    hv = torch.randn(3 * N, dtype=torch.float64).pin_memory()
    o1 = torch.empty(3 * N, dtype=torch.float64).pin_memory()
    f = lambda: L.check(lib.rq_apply_host(h, L.OP_QTILDE_V, hv.data_ptr(), o1.data_ptr(), 1))
    for _ in range(3): f()
    t0 = time.perf_counter()
    for _ in range(reps): f()
    return (time.perf_counter() - t0) / reps * 1e3
pos, off = ellipsoid_batch([4096] * 8, seed=1)
op = rq.MultiBodyOperator(rq.MultiBodyModel.from_arrays(pos, off))
for segs in (1, 8):
    os.environ["RQ_HOST_SEGS"] = str(segs); os.environ["RQ_HOST_SEG_MB"] = "1"
    print(f"tiny (8 bodies) segs {segs}: {timeit(op.plan.handle, int(off[-1]), 8):.3f} ms")
pos, off = make_config(2, seed=1000)
op = rq.MultiBodyOperator(rq.MultiBodyModel.from_arrays(pos, off))
for segs in (1, 2, 4, 8):
    os.environ["RQ_HOST_SEGS"] = str(segs); os.environ["RQ_HOST_SEG_MB"] = "2"
    print(f"cfg2 segs {segs}: {timeit(op.plan.handle, int(off[-1]), 1000, 10):.3f} ms")
