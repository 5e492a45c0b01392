"""Block-Krylov consumer (paper Eqs. 5-6) on the k = 32 multi-RHS kernels:
the constraint forces g from block CG on Q~ D Q~^T, the rigid-body velocities from Eq. 6,
checked against a dense solve built from the oracle's Q and against the original
formulation Q_Z D^{-1} Q_Z^T V = F (Eq. 4's first block row)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rq():
    import paper_1708_08427_b200 as rq
    from paper_1708_08427_b200 import _lib

    if _lib.device_count() < 1:
        pytest.fail("no GPU visible: the gpu tests must run on a B200 (no CPU fallback)")
    return rq


def test_block_cg_mobility_solve(rq, oracle_mod):
    import torch

    from paper_1708_08427_b200.krylov import DiagonalMobility, RigidBodyMobilitySolver
    from paper_1708_08427_b200.workloads import ellipsoid_batch

    counts = [200, 300, 150]
    pos, off = ellipsoid_batch(counts, seed=31)
    N, m, k = int(off[-1]), len(counts), 32
    op = rq.MultiBodyOperator(rq.MultiBodyModel.from_arrays(pos, off))
    rng = np.random.default_rng(32)
    d = rng.uniform(0.5, 2.0, size=3 * N)
    F = rng.normal(size=(6 * m, k))
    solver = RigidBodyMobilitySolver(op, DiagonalMobility(d))
    V, g, info = solver.solve(torch.from_numpy(F).cuda(), tol=1e-13)
    V, g = V.cpu().numpy(), g.cpu().numpy()
    assert info["relative_residual"] < 1e-13 and info["iterations"] < 200
    # dense reference from the oracle's Q = [Q_Z; Q~] per body
    QZ = np.zeros((6 * m, 3 * N))
    QT = np.zeros((3 * N - 6 * m, 3 * N))
    for j in range(m):
        n = counts[j]
        Qj = oracle_mod.OracleBody(pos[off[j]:off[j + 1]]).qv(np.eye(3 * n))
        cols = slice(3 * off[j], 3 * off[j + 1])
        QZ[6 * j:6 * j + 6, cols] = Qj[:6]
        r0 = 3 * off[j] - 6 * j
        QT[r0:r0 + 3 * n - 6, cols] = Qj[6:]
    D = np.diag(d)
    g_ref = -np.linalg.solve(QT @ D @ QT.T, QT @ D @ QZ.T @ F)
    V_ref = QZ @ D @ (QZ.T @ F + QT.T @ g_ref)
    assert np.linalg.norm(g - g_ref) / np.linalg.norm(g_ref) < 1e-10
    assert np.linalg.norm(V - V_ref) / np.linalg.norm(V_ref) < 1e-10
    # the original formulation: bead forces D^{-1} Q_Z^T V resolve to F
    lhs = QZ @ np.diag(1.0 / d) @ QZ.T @ V
    assert np.linalg.norm(lhs - F) / np.linalg.norm(F) < 1e-10
    # bead velocities are rigid-body motions: Q~ v = 0
    v = D @ (QZ.T @ F + QT.T @ g)
    assert np.abs(QT @ v).max() < 1e-10 * np.abs(v).max()
