"""Time the reference package as shipped (pure Python + numpy, imported from /root/reference in the
build container -- it does not travel to the GPU box) on a sample of config 2's bodies, next to the
C oracle on the same bodies and host.  SURVEY 8(d) CPU-baseline steps 1-3: single process as
shipped, and a multiprocessing pool over bodies.  Writes profiles/r02f_reference_python_timing.json.

  OPENBLAS_NUM_THREADS=1 python tools/ref_python_timing.py [n_bodies]
"""
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
from paper_1708_08427_b200.workloads import make_config  # noqa: E402

NB = int(sys.argv[1]) if len(sys.argv) > 1 else 8
pos, off = make_config(2, seed=1000, scale=NB / 1000.0)
n = int(off[1] - off[0])
bodies = [pos[off[j]:off[j + 1]] for j in range(len(off) - 1)]
rng = np.random.default_rng(0)
vs = [rng.normal(size=3 * len(b)) for b in bodies]
gs = [rng.normal(size=3 * len(b) - 6) for b in bodies]


def one_body(j):
    import rigidq  # the reference

    t0 = time.perf_counter()
    op = rigidq.BodyOperator(rigidq.BeadModel(bodies[j]))
    t_setup = time.perf_counter() - t0
    best = np.inf
    for _ in range(3):
        t0 = time.perf_counter()
        op.qtilde_v(vs[j])
        op.qtilde_tv(gs[j])
        best = min(best, time.perf_counter() - t0)
    return t_setup, best


if __name__ == "__main__":
    cores = len(os.sched_getaffinity(0))
    # (1) single process as shipped
    t0 = time.perf_counter()
    r = [one_body(j) for j in range(min(NB, 2))]
    single = {"bodies": len(r), "beads_per_body": n,
              "setup_beads_per_s": n * len(r) / sum(x[0] for x in r),
              "step_beads_per_s": n * len(r) / sum(x[1] for x in r),
              "step_s_per_body": float(np.mean([x[1] for x in r])), "setup_s_per_body": float(np.mean([x[0] for x in r]))}
    # (2) multiprocessing pool over bodies, one worker per core
    with mp.Pool(cores) as pool:
        t0 = time.perf_counter()
        r = pool.map(one_body, range(NB))
        wall = time.perf_counter() - t0
    # per-worker rates: every worker ran NB / cores bodies back to back
    pool_rate = cores * n / float(np.mean([x[1] for x in r]))
    pool_setup = cores * n / float(np.mean([x[0] for x in r]))
    # (3) the C oracle on the same bodies, all threads
    from oracle.oracle import OracleBatch

    t0 = time.perf_counter()
    ob = OracleBatch(pos, off, threads=cores)
    t_osetup = time.perf_counter() - t0
    v, g = np.concatenate(vs), np.concatenate(gs)
    best = np.inf
    for _ in range(5):
        t0 = time.perf_counter()
        ob.apply("qtilde_v", v)
        ob.apply("qtilde_tv", g)
        best = min(best, time.perf_counter() - t0)
    out = {"where": "build container (no GPU), %d cores" % cores, "config": "cfg2 bodies (4096-bead ellipsoid shells), %d bodies" % NB,
           "reference_python_single_process": single,
           "reference_python_pool": {"workers": cores, "step_beads_per_s": pool_rate, "setup_beads_per_s": pool_setup,
                                     "wall_s": wall, "note": "per-body min-of-3 step time inside each worker, x workers"},
           "c_oracle_all_threads": {"threads": cores, "step_beads_per_s": NB * n / best, "setup_beads_per_s": NB * n / t_osetup},
           }
    out["oracle_over_python_pool"] = out["c_oracle_all_threads"]["step_beads_per_s"] / pool_rate
    json.dump(out, open(os.path.join(ROOT, "profiles", "r02f_reference_python_timing.json"), "w"), indent=1)
    print(json.dumps(out, indent=1))
