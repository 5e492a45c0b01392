"""Phases of the numpy (pageable) host path on config 2: time for each rq_apply_host_async call
to return (input staging by host threads) and for the final rq_host_wait, per step of
Q~v + Q~^T g.  Run with RQ_HOST_THREADS=... to compare staging thread counts."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_08427_b200 as rq  # noqa: E402
from paper_1708_08427_b200 import _lib as L  # noqa: E402
from paper_1708_08427_b200._plan import host_result  # noqa: E402
from paper_1708_08427_b200.workloads import make_config  # noqa: E402

lib = L.lib()
pos, off = make_config(2, seed=1000)
N, m = int(off[-1]), len(off) - 1
op = rq.MultiBodyOperator(rq.MultiBodyModel.from_arrays(pos, off))
h = op.plan.handle
nv, ng = np.random.default_rng(0).normal(size=3 * N), np.random.default_rng(1).normal(size=3 * N - 6 * m)
pinned_out = os.environ.get("PROBE_PLAIN_OUT") is None
ph = []
for it in range(12):
    o1 = host_result(3 * N - 6 * m) if pinned_out else np.empty(3 * N - 6 * m)
    o2 = host_result(3 * N) if pinned_out else np.empty(3 * N)
    t0 = time.perf_counter()
    L.check(lib.rq_apply_host_async(h, L.OP_QTILDE_V, nv.ctypes.data, o1.ctypes.data, 1))
    t1 = time.perf_counter()
    L.check(lib.rq_apply_host_async(h, L.OP_QTILDE_TV, ng.ctypes.data, o2.ctypes.data, 1))
    t2 = time.perf_counter()
    L.check(lib.rq_host_wait(h))
    t3 = time.perf_counter()
    if it >= 2:
        ph.append((t1 - t0, t2 - t1, t3 - t2, t3 - t0))
a = np.median(np.array(ph), axis=0) * 1e3
print(f"threads={os.environ.get('RQ_HOST_THREADS', 'default')} pinned_out={pinned_out}: "
      f"stage1 {a[0]:.2f} ms, stage2 {a[1]:.2f} ms, wait {a[2]:.2f} ms, step {a[3]:.2f} ms", flush=True)
