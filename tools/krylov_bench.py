"""Block-CG mobility solve (paper Eqs. 5-6) on config-5 bodies with k = 32 right-hand sides:
iterations and time per iteration (two k = 32 multi-RHS applications + D)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1708_08427_b200 as rq  # noqa: E402
from paper_1708_08427_b200.krylov import DiagonalMobility, RigidBodyMobilitySolver  # noqa: E402
from paper_1708_08427_b200.workloads import ellipsoid_batch  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 200
pos, off = ellipsoid_batch([8192] * m, seed=1005)
N = int(off[-1])
op = rq.MultiBodyOperator(rq.MultiBodyModel.from_arrays(pos, off))
rng = np.random.default_rng(0)
solver = RigidBodyMobilitySolver(op, DiagonalMobility(rng.uniform(0.5, 2.0, size=3 * N)))
F = torch.from_numpy(rng.normal(size=(6 * m, 32))).cuda()
solver.solve(F, tol=1e-6, maxiter=3)
torch.cuda.synchronize()
t0 = time.perf_counter()
V, g, info = solver.solve(F, tol=1e-10)
torch.cuda.synchronize()
el = time.perf_counter() - t0
print({"bodies": m, "beads": N, "k": 32, **info, "seconds": el, "ms_per_iteration": el / info["iterations"] * 1e3,
       "bead_rhs_per_s_per_operator": 2 * info["iterations"] * N * 32 / el})
