"""Generate the golden fixtures that pin the oracle (and the GPU path) to the
reference package itself.

Runs ONLY in the build container, where the reference is importable:

    python tests/golden/make_golden.py

It imports /root/reference/pkg/src/rigidq, runs the reference on seeded
inputs, and writes tests/golden/*.npz.  The fixtures are committed; nothing
on the GPU box reads /root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import rigidq as R  # noqa: E402  (the reference package)

from paper_1708_08427_b200.workloads import ellipsoid_batch, sphere_shell  # noqa: E402

CASE_CODE = {R.NodeCase.LEAF: 0, R.NodeCase.BEAD_BEAD: 1, R.NodeCase.RIGID_BEAD: 2,
             R.NodeCase.GENERAL: 3}


def body_arrays(pos):
    model = R.BeadModel(pos)
    op = R.BodyOperator(model)
    tr, fa = op.tree, op.factors
    nodes = tr.nodes
    d = {}
    d["perm"] = np.asarray(tr.perm, np.int64)
    d["start"] = np.array([nd.start for nd in nodes], np.int64)
    d["stop"] = np.array([nd.stop for nd in nodes], np.int64)
    ch = np.array([nd.children if nd.children else (-1, -1) for nd in nodes], np.int64).reshape(-1, 2)
    d["left"], d["right"] = ch[:, 0].copy(), ch[:, 1].copy()
    d["split_axis"] = np.array([-1 if nd.split_axis is None else nd.split_axis for nd in nodes], np.int32)
    d["depth"] = np.array([nd.depth for nd in nodes], np.int32)
    d["centroid"] = np.array([nd.centroid for nd in nodes]).reshape(-1, 3)
    d["box"] = np.array([nd.box for nd in nodes]).reshape(-1, 2, 3)
    fs = fa.factors
    d["case"] = np.array([CASE_CODE[f.case] for f in fs], np.int32)
    d["fn"] = np.array([f.n for f in fs], np.int64)
    d["fnx"] = np.array([f.n_x for f in fs], np.int64)
    d["fny"] = np.array([f.n_y for f in fs], np.int64)
    d["swapped"] = np.array([f.swapped for f in fs], bool)
    d["t22"] = np.array([f.t22 for f in fs]).reshape(-1, 3, 3)
    om = [f.omega for f in fs]
    d["omega_k"] = np.array([0 if o is None else o.shape[0] for o in om], np.int32)
    d["omega"] = np.concatenate([o.ravel() for o in om if o is not None]) if any(
        o is not None for o in om) else np.zeros(0)
    d["res_offsets"] = np.asarray(fa.res_offsets, np.int64)
    d["total_rows"] = np.array(fa.total_rows, np.int64)
    return model, op, d


def multi_case(name, bodies, seed=0, k=3, with_z=False, with_q=False):
    rng = np.random.default_rng([seed, 99])
    counts = [b.shape[0] for b in bodies]
    offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    pos = np.concatenate(bodies)
    out = {"positions": pos, "offsets": offsets}
    models = []
    for j, b in enumerate(bodies):
        model, op, d = body_arrays(b)
        models.append(model)
        for key, val in d.items():
            out[f"b{j}_{key}"] = val
    mm = R.MultiBodyModel(models)
    mop = R.MultiBodyOperator(mm)
    N = int(offsets[-1])
    full, comp = 3 * N, 3 * N - 6 * len(bodies)
    small = min(counts) < 2
    v = rng.normal(size=full)
    w = rng.normal(size=full)
    out["v"], out["w"] = v, w
    out["qv"] = mop.apply("qv", v)
    out["qtv"] = mop.apply("qtv", w)
    V = rng.normal(size=(full, k))
    W = rng.normal(size=(full, k))
    out["V"], out["W"] = V, W
    out["qv_k"] = mop.apply("qv", V)
    out["qtv_k"] = mop.apply("qtv", W)
    if not small:
        out["qtilde_v"] = mop.apply("qtilde_v", v)
        out["qtilde_v_k"] = mop.apply("qtilde_v", V)
        # the reference raises ValueError on any length-0 block (matfree.py:92): n=2 bodies
        if min(counts) > 2:
            g = rng.normal(size=comp)
            G = rng.normal(size=(comp, k))
            out["g"], out["G"] = g, G
            out["qtilde_tv"] = mop.apply("qtilde_tv", g)
            out["qtilde_tv_k"] = mop.apply("qtilde_tv", G)
    if with_z:
        f = rng.normal(size=full)
        u = rng.normal(size=6 * len(bodies))
        zf, ztu = [], []
        for j, model in enumerate(models):
            z = R.assemble_z(model).entries
            zf.append(z @ f[3 * offsets[j]:3 * offsets[j + 1]])
            ztu.append(z.T @ u[6 * j:6 * j + 6])
        out["f"], out["u"] = f, u
        out["zf"], out["ztu"] = np.concatenate(zf), np.concatenate(ztu)
        out["model_centroid"] = np.array([m.centroid for m in models])
    if with_q:
        for j, model in enumerate(models):
            if model.n < 2:
                continue
            tree = R.build_tree(model)
            hq = R.generate_explicit_q(tree)
            out[f"q{j}_root_rows"] = hq.root_rows
            out[f"q{j}_block_node"] = np.array([b[0] for b in hq.blocks], np.int64)
            out[f"q{j}_block_col"] = np.array([b[1] for b in hq.blocks], np.int64)
            out[f"q{j}_block_rows"] = np.array([b[2].shape[0] for b in hq.blocks], np.int64)
            out[f"q{j}_block_data"] = np.concatenate([b[2].ravel() for b in hq.blocks]) if hq.blocks \
                else np.zeros(0)
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: m={len(bodies)} N={N} -> {os.path.getsize(path) / 1024:.0f} KiB")


def main():
    # SPEC.md:265/345/355 -- beads +-(0,0,1)
    multi_case("kat_pm", [np.array([[0.0, 0.0, 1.0], [0.0, 0.0, -1.0]])], with_z=True, with_q=True)
    # two beads, z split at the first ghost level
    multi_case("kat_two", [np.array([[0.1, 0.1, 0.1], [0.9, 0.9, 0.9]])], with_q=True)
    # BASELINE config 1 (CPU-runnable oracle case): sphere shell n=1024, seed 0
    multi_case("cfg1_sphere1024", [sphere_shell(1024, 0)], with_z=True)
    # config-2/4 style ellipsoid bodies of mixed size, including n=2 and n=3
    pos, off = ellipsoid_batch([2, 3, 50, 257, 1000, 513], seed=5)
    multi_case("ellipsoid_mix", [pos[off[j]:off[j + 1]] for j in range(len(off) - 1)], with_z=True)
    # reference cloud kinds (clouds.py) -- uniform, shell, lattice (beads on split planes)
    multi_case("uniform300", [R.make_cloud("uniform", 300, 3)], with_q=True)
    multi_case("grid500", [R.make_cloud("grid", 500, 0)], with_z=True)
    multi_case("shell700", [R.make_cloud("shell", 700, 1)])
    # a single-bead body next to normal ones (qv/qtv only; Q~ ops raise)
    multi_case("with_single", [np.array([[0.3, -0.2, 0.5]]), sphere_shell(40, 2)])
    # explicit Q (Algorithm 1) for validation sizes
    multi_case("explicit_q", [sphere_shell(64, 7), R.make_cloud("uniform", 33, 1)], with_q=True)
    # degenerate collinear input: parity only by span
    multi_case("line64", [R.make_cloud("line", 64, 0)])


if __name__ == "__main__":
    main()
