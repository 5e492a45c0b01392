"""Host-buffer application timeline on config 2 (pinned buffers): per-op time, plain vs pipelined."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_08427_b200 as rq  # noqa: E402
from paper_1708_08427_b200 import _lib as L  # noqa: E402
from paper_1708_08427_b200.workloads import make_config  # noqa: E402

lib = L.lib()
pos, off = make_config(2, seed=1000)
N, m = int(off[-1]), len(off) - 1
op = rq.MultiBodyOperator(rq.MultiBodyModel.from_arrays(pos, off))
h = op.plan.handle
hv = torch.randn(3 * N, dtype=torch.float64).pin_memory()
hg = torch.randn(3 * N - 6 * m, dtype=torch.float64).pin_memory()
o1 = torch.empty(3 * N - 6 * m, dtype=torch.float64).pin_memory()
o2 = torch.empty(3 * N, dtype=torch.float64).pin_memory()
fv = lambda: L.check(lib.rq_apply_host(h, L.OP_QTILDE_V, hv.data_ptr(), o1.data_ptr(), 1))  # noqa: E731
fg = lambda: L.check(lib.rq_apply_host(h, L.OP_QTILDE_TV, hg.data_ptr(), o2.data_ptr(), 1))  # noqa: E731
for mode in ("plain", "pipelined"):
    if mode == "plain":
        os.environ["RQ_HOST_PLAIN"] = "1"
    else:
        os.environ.pop("RQ_HOST_PLAIN", None)
    for name, f in (("qtilde_v", fv), ("qtilde_tv", fg)):
        for _ in range(3):
            f()
        t0 = time.perf_counter()
        for _ in range(10):
            f()
        print(f"{mode} {name}: {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms", flush=True)
os.environ["RQ_HOST_TRACE"] = "1"
fv()
fg()
