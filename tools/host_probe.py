"""Host-buffer application time on config 2: pinned / pageable, synchronous / queued pairs."""
import os
import sys
import time

import numpy as np
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
for pinned in (True, False):
    mk = (lambda t: t.pin_memory()) if pinned else (lambda t: t)
    hv = mk(torch.randn(3 * N, dtype=torch.float64))
    hg = mk(torch.randn(3 * N - 6 * m, dtype=torch.float64))
    o1 = mk(torch.empty(3 * N - 6 * m, dtype=torch.float64))
    o2 = mk(torch.empty(3 * N, dtype=torch.float64))

    def sync_step():
        L.check(lib.rq_apply_host(h, L.OP_QTILDE_V, hv.data_ptr(), o1.data_ptr(), 1))
        L.check(lib.rq_apply_host(h, L.OP_QTILDE_TV, hg.data_ptr(), o2.data_ptr(), 1))

    def async_step():
        L.check(lib.rq_apply_host_async(h, L.OP_QTILDE_V, hv.data_ptr(), o1.data_ptr(), 1))
        L.check(lib.rq_apply_host_async(h, L.OP_QTILDE_TV, hg.data_ptr(), o2.data_ptr(), 1))
        L.check(lib.rq_host_wait(h))

    for name, f in (("sync", sync_step), ("async pair", async_step)):
        for _ in range(3):
            f()
        t0 = time.perf_counter()
        for _ in range(10):
            f()
        print(f"{'pinned' if pinned else 'pageable'} {name}: {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms per step",
              flush=True)
nv, ng = np.random.default_rng(0).normal(size=3 * N), np.random.default_rng(1).normal(size=3 * N - 6 * m)
for _ in range(2):
    op.apply("qtilde_v", nv)
    op.apply("qtilde_tv", ng)
t0 = time.perf_counter()
for _ in range(5):
    op.apply("qtilde_v", nv)
    op.apply("qtilde_tv", ng)
print(f"numpy MultiBodyOperator.apply: {(time.perf_counter() - t0) / 5 * 1e3:.3f} ms per step")
