"""Digest of Q v / Q^T w / Q~ v / Q~^T g on mixed batches (small, config-2-like and one 2^20-bead
body): run before and after a kernel change that must keep results bit-identical and compare lines."""
import hashlib
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1708_08427_b200 as rq  # noqa: E402
from paper_1708_08427_b200.workloads import ellipsoid_batch, make_config  # noqa: E402

cases = {
    "mixed": ellipsoid_batch([300, 2, 1500, 77, 4096, 9000, 20000, 70000, 3, 129, 130, 257], seed=5),
    "cfg2x40": tuple(a for a in make_config(2, seed=11, scale=0.04)),
    "cfg3": tuple(a for a in make_config(3, seed=3, scale=0.25)),
}
for name, (pos, off) in cases.items():
    op = rq.MultiBodyOperator(rq.MultiBodyModel.from_arrays(pos, off))
    N, m = int(off[-1]), len(off) - 1
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    v = torch.randn(3 * N, generator=g, device="cuda", dtype=torch.float64)
    w = torch.randn(3 * N - 6 * m, generator=g, device="cuda", dtype=torch.float64)
    outs = []
    for opn, x in (("qv", v), ("qtv", v), ("qtilde_v", v)) + ((("qtilde_tv", w),) if int(np.diff(off).min()) > 2 else ()):
        y = op.apply(opn, x).cpu().numpy()
        outs.append(f"{opn}:{hashlib.sha1(y.tobytes()).hexdigest()[:12]}:{np.linalg.norm(y):.15e}")
    print(name, " ".join(outs))
