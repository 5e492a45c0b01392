"""Matrix-free Q / Q^T / Q~ / Q~^T (matfree.py:1-252 of the reference).

Every application runs on the B200 (rq_apply): a level-synchronous sweep of
chunk blobs streamed by TMA bulk copies plus a small per-body top tree.  The
public conventions are the reference's: vectors in ORIGINAL bead order,
shape (len,) or (len, k), 1-D in -> 1-D out, spectral layout [root 6 |
residues in postorder] (matfree.py:8-14), fresh output arrays, inputs never
mutated.  numpy inputs return numpy; contiguous float64 CUDA torch tensors
are used in place and return CUDA tensors (no host round trip).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from ._plan import Plan, _is_torch_cuda
from .errors import BodyTooSmallError, LengthMismatchError
from .factor import FactorTable, NodeCase, factor_all
from .model import BeadModel, MultiBodyModel
from .tree import BodyTree, build_tree

_MERGE_FLOPS = {NodeCase.BEAD_BEAD: 42, NodeCase.RIGID_BEAD: 114, NodeCase.GENERAL: 204}  # matfree.py:30
_CASE_CODE = {NodeCase.BEAD_BEAD: 1, NodeCase.RIGID_BEAD: 2, NodeCase.GENERAL: 3}


def _P(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def leaf_infoset(f) -> np.ndarray:
    """Info vector of a single bead: [f; 0] (matfree.py:33-38)."""
    f = np.asarray(f, dtype=float)
    m = np.zeros((6,) + f.shape[1:])
    m[:3] = f
    return m


def merge_infosets(factor, m_x, m_y):
    """One node's merge (matfree.py:41-62) on the GPU (rq_node_merge)."""
    m_x = np.asarray(m_x, dtype=float)
    m_y = np.asarray(m_y, dtype=float)
    shape = m_x.shape
    K = int(np.prod(shape[1:])) if m_x.ndim > 1 else 1
    mx = np.ascontiguousarray(m_x.reshape(6, K))
    my = np.ascontiguousarray(m_y.reshape(6, K))
    a, b = factor.ratios
    om = np.ascontiguousarray(factor.omega, dtype=float)
    rr = factor.residue_rows
    mp = np.empty((6, K))
    res = np.empty((max(rr, 1), K))
    L.check(L.lib().rq_node_merge(_CASE_CODE[factor.case], _P(om), float(a), float(b), _P(mx), _P(my), K,
                                  _P(mp), _P(res)))
    return mp.reshape(shape), res[:rr].reshape((rr,) + shape[1:])


def split_rvset(factor, l_p, res):
    """Adjoint of merge_infosets (matfree.py:65-83) on the GPU (rq_node_split)."""
    l_p = np.asarray(l_p, dtype=float)
    shape = l_p.shape
    K = int(np.prod(shape[1:])) if l_p.ndim > 1 else 1
    lp = np.ascontiguousarray(l_p.reshape(6, K))
    rr = factor.residue_rows
    r = np.zeros((max(rr, 1), K))
    if rr:
        r[:rr] = np.asarray(res, dtype=float).reshape(rr, K)
    a, b = factor.ratios
    om = np.ascontiguousarray(factor.omega, dtype=float)
    lx = np.empty((6, K))
    ly = np.empty((6, K))
    L.check(L.lib().rq_node_split(_CASE_CODE[factor.case], _P(om), float(a), float(b), _P(lp), _P(r), K,
                                  _P(lx), _P(ly)))
    return lx.reshape(shape), ly.reshape(shape)


def _as_columns(v, length, what="vector"):
    """matfree.py:86-92; also accepts CUDA torch tensors."""
    if _is_torch_cuda(v):
        import torch

        if v.shape[0] != length or v.dim() > 2:
            raise LengthMismatchError(f"{what} has shape {tuple(v.shape)}, expected ({length},) or ({length}, k)")
        if length == 0:
            raise ValueError(f"cannot reshape array of size 0 into shape ({length},newaxis)")
        v2 = v.reshape(length, -1).to(torch.float64).contiguous()
        return v2, v.dim() == 1
    v = np.asarray(v, dtype=float)
    if v.shape[0] != length or v.ndim > 2:
        raise LengthMismatchError(f"{what} has shape {v.shape}, expected ({length},) or ({length}, k)")
    return np.ascontiguousarray(v.reshape(length, -1)), v.ndim == 1


def _copy(x):
    return x.clone() if _is_torch_cuda(x) else x.copy()


def _plan_of(tree: BodyTree):
    return tree._plan


def upward_apply(tree: BodyTree, factors: FactorTable, v):
    """Q @ v in the spectral layout (Algorithm 2, matfree.py:95-121)."""
    n = tree.n
    v2, single = _as_columns(v, 3 * n)
    if n == 1:
        return _copy(v2[:, 0]) if single else _copy(v2)
    out = _plan_of(tree).apply("qv", v2)
    return out[:, 0] if single else out


def downward_apply(tree: BodyTree, factors: FactorTable, w):
    """Q.T @ w for a spectral-layout w (Algorithm 3, matfree.py:124-151)."""
    n = tree.n
    w2, single = _as_columns(w, 3 * n, "spectral vector")
    if n == 1:
        return _copy(w2[:, 0]) if single else _copy(w2)
    out = _plan_of(tree).apply("qtv", w2)
    return out[:, 0] if single else out


def qtilde_apply(tree: BodyTree, factors: FactorTable, v):
    """Complement rows only: Q~ v (matfree.py:154-158)."""
    if tree.n < 2:
        raise BodyTooSmallError("complement undefined for a single bead")
    v2, single = _as_columns(v, 3 * tree.n)
    out = _plan_of(tree).apply("qtilde_v", v2)
    return out[:, 0] if single else out


def qtilde_transpose_apply(tree: BodyTree, factors: FactorTable, g):
    """Q~^T g: downward pass seeded with a zero root vector (matfree.py:161-170)."""
    n = tree.n
    if n < 2:
        raise BodyTooSmallError("complement undefined for a single bead")
    g2, single = _as_columns(g, 3 * n - 6, "complement vector")
    out = _plan_of(tree).apply("qtilde_tv", g2)
    return out[:, 0] if single else out


class BodyOperator:
    """Fitted single-body operator (matfree.py:173-206)."""

    def __init__(self, model: BeadModel):
        self.model = model
        self.tree = build_tree(model)
        self.factors = factor_all(self.tree)

    @property
    def n(self) -> int:
        return self.tree.n

    def qv(self, v):
        return upward_apply(self.tree, self.factors, v)

    def qtv(self, w):
        return downward_apply(self.tree, self.factors, w)

    def qtilde_v(self, v):
        return qtilde_apply(self.tree, self.factors, v)

    def qtilde_tv(self, g):
        return qtilde_transpose_apply(self.tree, self.factors, g)

    def scipy_operator(self, complement: bool = False):
        from scipy.sparse.linalg import LinearOperator

        dim = 3 * self.n
        if complement:
            return LinearOperator((dim - 6, dim), matvec=self.qtilde_v, rmatvec=self.qtilde_tv)
        return LinearOperator((dim, dim), matvec=self.qv, rmatvec=self.qtv)


_OP_NAMES = ("qv", "qtv", "qtilde_v", "qtilde_tv")  # matfree.py:209


class _BodyViews:
    """Per-body BodyOperator views, built on first access (reference attribute
    MultiBodyOperator.bodies, matfree.py:219-221)."""

    def __init__(self, model):
        self._model = model
        self._cache = {}

    def __len__(self):
        return self._model.m

    def __getitem__(self, j):
        if j < 0:
            j += len(self)
        if j not in self._cache:
            self._cache[j] = BodyOperator(self._model.bodies[j])
        return self._cache[j]

    def __iter__(self):
        return (self[j] for j in range(len(self)))


class MultiBodyOperator:
    """Block-diagonal operator over an ordered set of bodies (matfree.py:212-247).

    All bodies share ONE device plan: a single batched setup and one fused
    launch sequence per application, whatever the number of bodies.  Outputs
    equal the concatenation of per-body runs bit-exactly (per-body arithmetic
    never depends on the batch).
    """

    def __init__(self, model: MultiBodyModel, max_depth: int = 96):
        self.model = model
        self.plan = Plan(model.positions, model.offsets, max_depth=max_depth)
        self.bodies = _BodyViews(model)
        self._n = np.diff(model.offsets)
        self._N = int(model.offsets[-1])
        self._min_n = int(self._n.min())

    def _lengths(self, op: str):
        """Total (input, output) lengths of the concatenated per-body blocks (matfree.py:223-233);
        per-call host work is O(1) in the number of bodies (min body size cached)."""
        full = 3 * self._N
        if op in ("qv", "qtv"):
            return full, full
        if self._min_n < 2:
            raise BodyTooSmallError("complement operators need every body to have >= 2 beads")
        comp = full - 6 * len(self._n)
        return (full, comp) if op == "qtilde_v" else (comp, full)

    def apply(self, op: str, v):
        if op not in _OP_NAMES:
            raise ValueError(f"op must be one of {_OP_NAMES}, got {op!r}")
        in_len, out_len = self._lengths(op)
        v2, single = _as_columns(v, in_len)
        if op == "qtilde_tv" and self._min_n == 2:
            # the reference applies each body block separately and a length-0
            # block fails its reshape (matfree.py:92, 245): kept as-is
            raise ValueError("cannot reshape array of size 0 into shape (0,newaxis)")
        out = self.plan.apply(op, v2)
        return out[:, 0] if single else out

    def apply_many(self, items):
        """Several host (numpy) applications at once: ``[(op, v), ...] -> [result, ...]``.
        Same results as ``[self.apply(op, v) for op, v in items]``; the applications are queued
        together so consecutive host<->device copies overlap (rq_apply_host_async)."""
        prepared = []
        for op, v in items:
            if op not in _OP_NAMES:
                raise ValueError(f"op must be one of {_OP_NAMES}, got {op!r}")
            if _is_torch_cuda(v):
                raise TypeError("apply_many takes host (numpy) vectors; use apply for CUDA tensors")
            if op == "qtilde_tv" and self._min_n == 2:
                raise ValueError("cannot reshape array of size 0 into shape (0,newaxis)")
            in_len, _ = self._lengths(op)
            v2, single = _as_columns(v, in_len)
            prepared.append((op, v2, single))
        outs = self.plan.apply_host_many([(op, v2) for op, v2, _ in prepared])
        return [o[:, 0] if single else o for o, (_, _, single) in zip(outs, prepared)]

    def zf(self, f, origin=None):
        """Per-body [sum f; sum (r - c) x f] (6m,) -- Z @ f without assembling Z."""
        f2, single = _as_columns(f, 3 * self.model.n_total, "force vector")
        out = self.plan.z(L.Z_F, f2, origin)
        return out[:, 0] if single else out

    def ztu(self, u, origin=None):
        """Per-bead V + w x (r - c) (3N,) -- Z.T @ u without assembling Z."""
        u2, single = _as_columns(u, 6 * self.model.m, "rigid-body vector")
        out = self.plan.z(L.Z_TU, u2, origin)
        return out[:, 0] if single else out


def multibody_apply(model: MultiBodyModel, op: str, v):
    """One-shot block-diagonal application (matfree.py:250-252)."""
    return MultiBodyOperator(model).apply(op, v)
