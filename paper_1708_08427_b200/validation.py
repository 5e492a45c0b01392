"""Dense validation tools of the reference (oracle.py:26-270) on the GPU.

The reference checks its hierarchical Q against a dense complement of Z's row space
(SVD) and reports orthogonality quality per body.  Here the dense linear algebra runs
on the GPU (cuSOLVER SVD and cuBLAS through torch) and the operators are the B200 ones:

  dense_complement(z, guard)       oracle.py:38-47  trailing right singular vectors of Z
  projector_distance(a, b)         oracle.py:50-58  max |A^T A - B^T B| (row spaces)
  max_abs_gram_deviation(q, block) oracle.py:208-217
  body_report(model, seed, guard)  oracle.py:220-244
  report_to_csv(rows)              oracle.py:261-270 (byte-stable rendering)

Not provided: the naive divide-and-conquer of the paper's §2.2 (``naive_divide_conquer``,
a deliberately unstable classical Gram-Schmidt baseline) and ``orthogonality_report``,
which draws its bodies from the reference's cloud kinds (clouds.py, out of scope).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ShapeMismatchError, SizeGuardError


def _dev(x):
    import torch

    return torch.as_tensor(np.asarray(x, dtype=float), device="cuda")


@dataclass(frozen=True)
class DenseComplement:
    """Orthonormal rows spanning the complement of the resultant row space."""

    qtilde: np.ndarray
    rank: int  # numerical rank of Z (5 for collinear bodies, else 6)


def dense_complement(z, guard: int = 6000) -> DenseComplement:
    """Full orthogonal decomposition of Z (cuSOLVER SVD); the trailing directions span the
    complement.  Rank deficiency (collinear bodies) widens the complement."""
    import torch

    entries = z.entries if hasattr(z, "entries") else np.asarray(z, dtype=float)
    if entries.shape[1] > guard:
        raise SizeGuardError(f"3n = {entries.shape[1]} exceeds guard {guard}")
    _, s, vt = torch.linalg.svd(_dev(entries), full_matrices=True)
    s = s.cpu().numpy()
    tol = max(entries.shape) * np.finfo(float).eps * (s[0] if s.size else 0.0)
    rank = int((s > tol).sum())
    return DenseComplement(vt[rank:].cpu().numpy(), rank)


def projector_distance(a, b) -> float:
    """Entrywise max difference of the projectors onto two row spaces; zero iff the spaces
    coincide (rows themselves need not match)."""
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    if a.shape[1] != b.shape[1]:
        raise ShapeMismatchError(f"column counts differ: {a.shape[1]} vs {b.shape[1]}")
    if a.size == 0 and b.size == 0:
        return 0.0
    ta, tb = _dev(a), _dev(b)
    d = ta.T @ ta - tb.T @ tb
    return float(d.abs().max()) if d.numel() else 0.0


def max_abs_gram_deviation(q, block: int = 768) -> float:
    """max |Q Q^T - I| computed in row blocks on the GPU."""
    tq = _dev(q)
    worst = 0.0
    m = tq.shape[0]
    for i0 in range(0, m, block):
        g = tq[i0:i0 + block] @ tq.T
        rows = g.shape[0]
        g[range(rows), [i0 + r for r in range(rows)]] -= 1.0
        worst = max(worst, float(g.abs().max()))
    return worst


REPORT_COLUMNS = ("n", "qqt", "qtq", "qv_dev", "qtv_dev", "roundtrip_qtq", "roundtrip_qqt")


def body_report(model, seed: int = 0, dense_guard: int = 6000) -> dict:
    """One orthogonality-quality row for a single body (None = skipped), oracle.py:220-244:
    the explicit Q (Algorithm 1) against the matrix-free applications and their round trips."""
    from .factor import factor_all, generate_explicit_q
    from .matfree import downward_apply, upward_apply
    from .tree import build_tree

    n = model.n
    row = {c: None for c in REPORT_COLUMNS}
    row["n"] = n
    if n < 2:
        return row
    tree = build_tree(model)
    factors = factor_all(tree)
    hq = generate_explicit_q(tree, factors)
    rng = np.random.default_rng([seed, n])
    v = rng.normal(size=3 * n)
    w = rng.normal(size=3 * n)
    if 3 * n <= dense_guard:
        qd = hq.to_dense("tree")
        row["qqt"] = max_abs_gram_deviation(qd)
        row["qtq"] = max_abs_gram_deviation(qd.T)
    up = upward_apply(tree, factors, v)
    down = downward_apply(tree, factors, w)
    row["qv_dev"] = float(np.abs(hq.matvec(v) - up).max())
    row["qtv_dev"] = float(np.abs(hq.rmatvec(w) - down).max())
    row["roundtrip_qtq"] = float(np.abs(downward_apply(tree, factors, up) - v).max())
    row["roundtrip_qqt"] = float(np.abs(upward_apply(tree, factors, down) - w).max())
    return row


def report_to_csv(rows) -> str:
    """Render report rows byte-stably; skipped cells become 'na'."""
    lines = [",".join(REPORT_COLUMNS)]
    for row in rows:
        cells = [str(row["n"])]
        cells += ["na" if row[c] is None else f"{row[c]:.17e}" for c in REPORT_COLUMNS[1:]]
        lines.append(",".join(cells))
    return "\n".join(lines) + "\n"
