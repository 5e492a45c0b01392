"""Block-Krylov consumer of the complement operators (arxiv 1708.08427).

For rigid bodies in a mobility problem with a symmetric positive-definite bead mobility D,
the paper replaces the dense D^{-1} of Z D^{-1} Z^T V = F by the orthogonal basis
Q = [Q_Z; Q~] of each body (Q_Z: orthonormal rows spanning Z's row space):

    Q~ D Q~^T g = - Q~ D Q_Z^T F^         (Eq. 5: constraint forces g, by a Krylov method)
    V = Q_Z D (Q_Z^T F^ + Q~^T g)         (Eq. 6: rigid-body velocities)

where F^ are the 6 resultants per body in the Q_Z coordinates.  Here both are solved for a
block of k right-hand sides with block conjugate gradients (O'Leary 1980); every iteration
applies Q~^T and Q~ to a (rows, k) block -- the multi-RHS kernels (k_mrhs, rq_mrhs.cu) with
k = 32 -- and D.  Q_Z and Q~ are the root rows and the residue rows of the full hierarchical Q
of matfree.py:95-151 (the Q layout: per body [6 root rows | 3n - 6 residue rows]), so
Q_Z^T F^ + Q~^T g is one Q^T application and Q_Z D (...) the root rows of one Q application.

D is the caller's (the paper uses a fast multipole method); ``DiagonalMobility`` is a simple
symmetric positive-definite stand-in (a positive weight per bead coordinate).
"""

from __future__ import annotations

import numpy as np


class DiagonalMobility:
    """D = diag(d), d > 0 per bead coordinate (3N,): a symmetric positive-definite mobility."""

    def __init__(self, d):
        import torch

        self.d = torch.as_tensor(d, dtype=torch.float64, device="cuda").reshape(-1, 1)
        if bool((self.d <= 0).any()):
            raise ValueError("mobility weights must be positive")

    def __call__(self, x):
        return self.d * x


def block_cg(apply_a, b, tol: float = 1e-12, maxiter: int = 500):
    """Block conjugate gradients for A X = B, A symmetric positive definite (torch, (n, k)).

    The search block is re-orthonormalised every iteration (shifted Cholesky-QR: one k x k
    Gram matrix, a Cholesky factor and a triangular solve, so it stays one GEMM-sized pass over
    the block), so the k x k systems stay symmetric positive definite when columns converge at
    different rates (the plain O'Leary recurrence breaks down on the rank-deficient residual
    block).  Returns (X, iterations, largest relative residual over the columns).
    """
    import torch

    def orth(w):
        gram = w.T @ w
        shift = 1e-14 * float(torch.trace(gram)) / gram.shape[0] + 1e-300
        c = torch.linalg.cholesky(gram + shift * torch.eye(gram.shape[0], dtype=w.dtype, device=w.device))
        return torch.linalg.solve_triangular(c.T, w, upper=True, left=False)  # w C^{-T}

    x = torch.zeros_like(b)
    r = b.clone()
    bnorm = torch.linalg.vector_norm(b, dim=0).clamp_min(1e-300)
    p = orth(r)
    res = torch.linalg.vector_norm(r, dim=0) / bnorm
    it = 0
    for it in range(1, maxiter + 1):
        q = apply_a(p)
        pap = p.T @ q
        alpha = torch.linalg.solve(pap, p.T @ r)
        x = x + p @ alpha
        r = r - q @ alpha
        res = torch.linalg.vector_norm(r, dim=0) / bnorm
        if float(res.max()) < tol:
            break
        beta = -torch.linalg.solve(pap, q.T @ r)  # next direction A-conjugate to this block
        p = orth(r + p @ beta)
    return x, it, res


class RigidBodyMobilitySolver:
    """Eqs. (5)-(6) of the paper for a MultiBodyOperator and a mobility D (callable on
    (3N, k) CUDA blocks).  ``solve(F)`` takes the 6 resultants per body in the Q_Z
    coordinates, (6m, k) on the GPU, and returns (V (6m, k), g (3N - 6m, k), info)."""

    def __init__(self, op, mobility):
        import torch

        self.op = op
        self.D = mobility
        n = np.asarray(op.model.offsets, dtype=np.int64)
        self.N, self.m = int(n[-1]), len(n) - 1
        if np.any(np.diff(n) < 2):
            raise ValueError("every body needs >= 2 beads (the complement has 3n - 6 rows)")
        b0 = 3 * n[:-1]
        root = (b0[:, None] + np.arange(6)[None, :]).reshape(-1)
        comp = np.concatenate([b0[j] + 6 + np.arange(3 * (n[j + 1] - n[j]) - 6) for j in range(self.m)])
        self.root = torch.as_tensor(root, device="cuda")
        self.comp = torch.as_tensor(comp, device="cuda")

    def _q_layout(self, f_root, g):
        import torch

        k = f_root.shape[1]
        x = torch.zeros((3 * self.N, k), dtype=torch.float64, device="cuda")
        x[self.root] = f_root
        if g is not None:
            x[self.comp] = g
        return x

    def apply_schur(self, g):
        """Q~ D Q~^T g (the operator of Eq. 5)."""
        return self.op.apply("qtilde_v", self.D(self.op.apply("qtilde_tv", g)))

    def solve(self, f_root, tol: float = 1e-12, maxiter: int = 500):
        f_root = f_root.reshape(6 * self.m, -1)
        dqzf = self.D(self.op.apply("qtv", self._q_layout(f_root, None)))  # D Q_Z^T F^
        rhs = -self.op.apply("qtilde_v", dqzf)                             # Eq. 5 right-hand side
        g, iters, res = block_cg(self.apply_schur, rhs, tol=tol, maxiter=maxiter)
        w = self.D(self.op.apply("qtv", self._q_layout(f_root, g)))      # D (Q_Z^T F^ + Q~^T g)
        v = self.op.apply("qv", w)[self.root]                             # Eq. 6: Q_Z (...)
        return v, g, {"iterations": iters, "relative_residual": float(res.max())}
