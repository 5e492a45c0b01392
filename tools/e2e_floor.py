"""Copy-only floor of the pipelined host-buffer apply: the same H2D / D2H byte counts and
segment structure as rq_apply_host on config 2, without kernels, vs the real call."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_08427_b200 as rq  # noqa: E402
from paper_1708_08427_b200 import _lib as L  # noqa: E402
from paper_1708_08427_b200.workloads import make_config  # noqa: E402

pos, off = make_config(2, seed=1000)
N, m = int(off[-1]), len(off) - 1
op = rq.MultiBodyOperator(rq.MultiBodyModel.from_arrays(pos, off))
h, lib = op.plan.handle, L.lib()
hv = torch.randn(3 * N, dtype=torch.float64).pin_memory()
o1 = torch.empty(3 * N, dtype=torch.float64).pin_memory()
d_in = torch.empty(3 * N, dtype=torch.float64, device="cuda")
d_out = torch.empty(3 * N, dtype=torch.float64, device="cuda")
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()

def copies(nseg):
    seg = (3 * N + nseg - 1) // nseg
    evs = []
    for i in range(nseg):
        with torch.cuda.stream(s_in):
            d_in[i * seg:(i + 1) * seg].copy_(hv[i * seg:(i + 1) * seg], non_blocking=True)
            e = torch.cuda.Event(); e.record(s_in); evs.append(e)
    for i in range(nseg):
        s_out.wait_event(evs[i])
        with torch.cuda.stream(s_out):
            o1[i * seg:(i + 1) * seg].copy_(d_out[i * seg:(i + 1) * seg], non_blocking=True)
    s_out.synchronize()

def real():
    L.check(lib.rq_apply_host(h, L.OP_QTILDE_V, hv.data_ptr(), o1.data_ptr(), 1))

for name, fn in (("copies x8", lambda: copies(8)), ("copies x16", lambda: copies(16)), ("copies x1", lambda: copies(1)), ("rq_apply_host Q~v", real)):
    for _ in range(3):
        fn()
    t0 = time.perf_counter()
    for _ in range(20):
        fn()
    print(f"{name:22s} {(time.perf_counter() - t0) / 20 * 1e3:.3f} ms")
