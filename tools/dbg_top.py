import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1708_08427_b200 as rq
from oracle import oracle as O
from paper_1708_08427_b200.workloads import ellipsoid_batch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 50000
pos, off = ellipsoid_batch([n], seed=11)
op = rq.MultiBodyOperator(rq.MultiBodyModel.from_arrays(pos, off))
print(op.plan.info()["top_global"], op.plan.info()["top_staged"])
ref = O.OracleBatch(pos, off, threads=8)
v = np.random.default_rng(5).normal(size=3 * n)
a = op.apply("qv", v)
b = ref.apply("qv", v)
d = np.abs(a - b) > 1e-9 * np.abs(b).max()
print("root rows bad:", d[:6].sum(), "bad rows:", d.sum(), "of", len(d))
idx = np.nonzero(d)[0]
print(idx[:20], idx[-20:])
f = op.plan.export_factors(0)
ro = f["res_offsets"]
cs = f["case"]
n_ = f["n"]
bad_nodes = set()
for r in idx[:2000]:
    k = np.searchsorted(ro, r, side="right") - 1
    bad_nodes.add(int(k))
bn = sorted(bad_nodes)
print("bad nodes", len(bn), [(k, int(cs[k]), int(n_[k])) for k in bn[:30]])
g = np.random.default_rng(6).normal(size=3 * n)
a2 = op.apply("qtv", g)
b2 = ref.apply("qtv", g)
print("qtv rel", np.linalg.norm(a2 - b2) / np.linalg.norm(b2))
t = op.plan.export_tree(0)
L = t["stop"] - t["start"]
lo = [k for k in bn if k >= 0]
badset = set(lo)
for k in lo[:12]:
    l, r = int(t["left"][k]), int(t["right"][k])
    print(k, "n", L[k], "children", (l, int(L[l]), l in badset), (r, int(L[r]), r in badset), "case", int(cs[k]), "swapped", int(f["swapped"][k]))
