"""Small end-to-end run of every kernel family: wave sweeps, staged and dataflow top trees,
Q / Q^T layout passes, the multi-RHS kernels (units and level-parallel tops), Z ops, the
host-buffer path.  Run against librigidq_b200_check.so (RQ_LIB_PATH, device-side bounds and
staging-phase asserts) by tests/test_gpu_checks.py; outputs go to argv[1] (.npz) so the
test can compare them with the product library's."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_08427_b200 as rq  # noqa: E402
from paper_1708_08427_b200.workloads import ellipsoid_batch, sphere_shell  # noqa: E402

os.environ.setdefault("RQ_WAVE_ROUNDS", "3")
counts = [4096] * 6 + [2, 3, 130, 700, 70000]  # the 70000-bead body: dataflow top tree
pos, off = ellipsoid_batch(counts, seed=3)
op = rq.MultiBodyOperator(rq.MultiBodyModel.from_arrays(pos, off))
N, m = int(off[-1]), len(off) - 1
rng = np.random.default_rng(0)
v = torch.from_numpy(rng.normal(size=3 * N)).cuda()
res = {}
for name in ("qv", "qtv", "qtilde_v"):
    res[name] = op.apply(name, v).cpu().numpy()
keep = [j for j in range(m) if counts[j] >= 3]
pos2 = np.concatenate([pos[off[j]:off[j + 1]] for j in keep])
off2 = np.concatenate([[0], np.cumsum([counts[j] for j in keep])])
op2 = rq.MultiBodyOperator(rq.MultiBodyModel.from_arrays(pos2, off2))
g = torch.from_numpy(rng.normal(size=3 * int(off2[-1]) - 6 * len(keep))).cuda()
res["qtilde_tv"] = op2.apply("qtilde_tv", g).cpu().numpy()
V = torch.from_numpy(rng.normal(size=(3 * N, 40))).cuda()
res["qv_k40"] = op.apply("qv", V).cpu().numpy()
res["qtv_k40"] = op.apply("qtv", V).cpu().numpy()
big = sphere_shell(70000, 1)
op3 = rq.MultiBodyOperator(rq.MultiBodyModel.from_arrays(big, np.array([0, 70000])))
V3 = torch.from_numpy(rng.normal(size=(3 * 70000, 33))).cuda()
G3 = op3.apply("qtilde_v", V3)
res["big_qtilde_v_k33"] = G3.cpu().numpy()
res["big_qtilde_tv_k33"] = op3.apply("qtilde_tv", G3).cpu().numpy()
res["zf"] = op.zf(v).cpu().numpy()
res["ztu"] = op.ztu(torch.from_numpy(rng.normal(size=6 * m)).cuda()).cpu().numpy()
res["host_qtilde_v"] = op.apply("qtilde_v", v.cpu().numpy())
torch.cuda.synchronize()
if len(sys.argv) > 1:
    np.savez(sys.argv[1], **res)
print("sanitize run ok")
