"""Parity at the full BASELINE.json sizes: the CUDA path vs the C oracle (pinned to the
reference by tests/golden) on the same seeded inputs, per body, 1e-12 relative in
fp64 (north_star), and exact tree / index layout.

  config 1  1 x 1024 sphere shell: dense Q~ from the operator itself,
            ||Q~ Q~^T - I||, ||Z Q~^T||, and the dense Q~ vs the oracle's
  config 2  1000 x 4096 ellipsoid shells: Q~v and Q~^T g per body (all bodies)
  config 3  1 x 2^20 sphere shell: exported tree / factor layout equal to the
            oracle's (perm, start, stop, children, split axis, depth, box, centroid,
            case, n_x, n_y, swapped, res_offsets) and all four operators
  config 4  the heterogeneous generator (log-uniform n in [500, 50000]) at 1/10 of
            the body count, 500 bodies stratified by size incl. the largest: Q~v,
            Q~^T g, Zf, Z^T u per body
  config 5  200 x 8192 bodies with k = 32 right-hand sides: Q~V, Q~^T G per body and
            column
"""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-12
THREADS = len(os.sched_getaffinity(0))


@pytest.fixture(scope="module")
def rq():
    import paper_1708_08427_b200 as rq
    from paper_1708_08427_b200 import _lib

    if _lib.device_count() < 1:
        pytest.fail("no GPU visible: the gpu tests must run on a B200 (no CPU fallback)")
    return rq


def per_body_worst(out, ref, lens):
    """max over bodies (and columns) of ||out - ref||_2 / ||ref||_2 on each body's block."""
    out = np.asarray(out).reshape(len(ref), -1)
    ref = np.asarray(ref).reshape(len(ref), -1)
    starts = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
    keep = np.asarray(lens) > 0
    d2 = np.add.reduceat((out - ref) ** 2, starts, axis=0)[keep]
    r2 = np.add.reduceat(ref ** 2, starts, axis=0)[keep]
    return float(np.sqrt(d2 / np.maximum(r2, 1e-300)).max())


def _dev(op, name, x):
    import torch

    return op.apply(name, torch.from_numpy(np.ascontiguousarray(x)).cuda()).cpu().numpy()


def test_config1_dense_invariants(rq, oracle_mod):
    from paper_1708_08427_b200.workloads import make_config

    pos, off = make_config(1, seed=0)
    n = int(off[-1])
    op = rq.MultiBodyOperator(rq.MultiBodyModel.from_arrays(pos, off))
    I = np.eye(3 * n - 6)
    qt_t = _dev(op, "qtilde_tv", I)            # Q~^T, (3n, 3n-6): column c = Q~^T e_c
    qq = _dev(op, "qtilde_v", qt_t)            # Q~ Q~^T
    assert np.abs(qq - I).max() < 1e-12
    z = rq.assemble_z(rq.BeadModel(pos)).entries  # dense 6 x 3n about the centroid (model.py:129-149)
    assert np.abs(z @ qt_t).max() < 1e-12 * np.abs(z).max()
    ref = oracle_mod.OracleBatch(pos, off, threads=1).apply("qtilde_tv", I)
    assert np.abs(qt_t - ref).max() < 1e-12


def test_config2_full_per_body(rq, oracle_mod):
    from paper_1708_08427_b200.workloads import make_config

    pos, off = make_config(2, seed=1000)
    n = np.diff(off)
    m = len(n)
    op = rq.MultiBodyOperator(rq.MultiBodyModel.from_arrays(pos, off))
    ref = oracle_mod.OracleBatch(pos, off, threads=THREADS)
    rng = np.random.default_rng(20)
    v = rng.normal(size=3 * int(off[-1]))
    g = rng.normal(size=3 * int(off[-1]) - 6 * m)
    assert per_body_worst(_dev(op, "qtilde_v", v), ref.apply("qtilde_v", v), 3 * n - 6) < TOL
    assert per_body_worst(_dev(op, "qtilde_tv", g), ref.apply("qtilde_tv", g), 3 * n) < TOL


def test_config3_full_tree_and_operators(rq, oracle_mod):
    from paper_1708_08427_b200.workloads import make_config

    pos, off = make_config(3, seed=0)
    n = int(off[-1])
    assert n == 1 << 20
    op = rq.MultiBodyOperator(rq.MultiBodyModel.from_arrays(pos, off))
    ob = oracle_mod.OracleBody(pos)
    a = op.plan.export_tree(0)
    for key in ("perm", "start", "stop", "left", "right", "split_axis", "depth"):
        np.testing.assert_array_equal(a[key], getattr(ob, key), err_msg=key)
    np.testing.assert_array_equal(a["box"], ob.box)
    np.testing.assert_array_equal(a["centroid"], ob.centroid)
    f = op.plan.export_factors(0, omega=False)
    for key, ok in (("case", "case"), ("n", "fn"), ("nx", "fnx"), ("ny", "fny"), ("res_offsets", "res_offsets")):
        np.testing.assert_array_equal(f[key], getattr(ob, ok), err_msg=key)
    np.testing.assert_array_equal(f["swapped"].astype(bool), ob.swapped)
    assert f["total_rows"] == ob.total_rows == 3 * n
    np.testing.assert_allclose(f["t22"], ob.t22, rtol=0, atol=1e-12)
    rng = np.random.default_rng(30)
    v = rng.normal(size=3 * n)
    g = rng.normal(size=3 * n - 6)
    for name, x in (("qv", v), ("qtv", v), ("qtilde_v", v), ("qtilde_tv", g)):
        out, ref = _dev(op, name, x), getattr(ob, name)(x)
        assert np.linalg.norm(out - ref) / np.linalg.norm(ref) < TOL, name


def test_config4_stratified_sample(rq, oracle_mod):
    from paper_1708_08427_b200.workloads import make_config

    pos, off = make_config(4, seed=1000, scale=0.1)
    n = np.diff(off)
    m = len(n)
    op = rq.MultiBodyOperator(rq.MultiBodyModel.from_arrays(pos, off))
    rng = np.random.default_rng(40)
    N = int(off[-1])
    v = rng.normal(size=3 * N)
    g = rng.normal(size=3 * N - 6 * m)
    f = rng.normal(size=3 * N)
    u = rng.normal(size=6 * m)
    yv, yg = _dev(op, "qtilde_v", v), _dev(op, "qtilde_tv", g)
    import torch

    zf = op.zf(torch.from_numpy(f).cuda()).cpu().numpy()
    ztu = op.ztu(torch.from_numpy(u).cuda()).cpu().numpy()
    order = np.argsort(n, kind="stable")
    pick = np.unique(np.concatenate([order[np.linspace(0, m - 1, 490).astype(int)], order[-10:]]))
    pos_s = np.concatenate([pos[off[j]:off[j + 1]] for j in pick])
    off_s = np.concatenate([[0], np.cumsum(n[pick])])
    ref = oracle_mod.OracleBatch(pos_s, off_s, threads=THREADS)
    full_rows = lambda x, w: np.concatenate([x[w * off[j]:w * off[j + 1]] for j in pick])  # noqa: E731
    comp0 = 3 * off[:-1] - 6 * np.arange(m)
    comp_rows = lambda x: np.concatenate([x[comp0[j]:comp0[j] + 3 * n[j] - 6] for j in pick])  # noqa: E731
    ns = n[pick]
    assert per_body_worst(comp_rows(yv), ref.apply("qtilde_v", full_rows(v, 3)), 3 * ns - 6) < TOL
    assert per_body_worst(full_rows(yg, 3), ref.apply("qtilde_tv", comp_rows(g)), 3 * ns) < TOL
    zf_s = np.concatenate([zf[6 * j:6 * j + 6] for j in pick])
    zref = ref.zf(full_rows(f, 3))
    # Zf normalised by ||Z||_F ||f||_2 per body (random forces cancel in the sums):
    # ||Z||_F^2 = 3n + 2 sum_k |r_k - c|^2 (identity blocks and skew(r_k - c) blocks)
    for i, j in enumerate(pick):
        p = pos[off[j]:off[j + 1]]
        zfro = np.sqrt(3 * n[j] + 2 * ((p - p.mean(0)) ** 2).sum())
        scale = zfro * np.linalg.norm(f[3 * off[j]:3 * off[j + 1]])
        assert np.abs(zf_s[6 * i:6 * i + 6] - zref[6 * i:6 * i + 6]).max() < TOL * scale
    u_s = np.concatenate([u[6 * j:6 * j + 6] for j in pick])
    assert per_body_worst(full_rows(ztu, 3), ref.ztu(u_s), 3 * ns) < TOL


def test_config5_multi_rhs(rq, oracle_mod):
    from paper_1708_08427_b200.workloads import ellipsoid_batch

    pos, off = ellipsoid_batch([8192] * 200, seed=1005)
    n = np.diff(off)
    m = len(n)
    op = rq.MultiBodyOperator(rq.MultiBodyModel.from_arrays(pos, off))
    ref = oracle_mod.OracleBatch(pos, off, threads=THREADS)
    rng = np.random.default_rng(50)
    V = rng.normal(size=(3 * int(off[-1]), 32))
    G = rng.normal(size=(3 * int(off[-1]) - 6 * m, 32))
    assert per_body_worst(_dev(op, "qtilde_v", V), ref.apply("qtilde_v", V), 3 * n - 6) < TOL
    assert per_body_worst(_dev(op, "qtilde_tv", G), ref.apply("qtilde_tv", G), 3 * n) < TOL
