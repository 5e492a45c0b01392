"""Bead-cloud inputs and the Z (force/torque resultant) operators.

Mirrors model.py of the reference (BeadModel / MultiBodyModel / ZMatrix /
assemble_z / centroid / skew, model.py:25-149).  The duplicate-bead check of
model.py:65-78 runs on the GPU (hash grid, rq_check_duplicates); the Zf /
Z^T u contractions run on the GPU without assembling Z (rq_z_apply).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from ._plan import check_duplicates as _gpu_check_duplicates
from .errors import DuplicateBeadsError

DUP_TOL_FACTOR = 1e-12  # model.py:22


def skew(r) -> np.ndarray:
    """Return the 3x3 matrix A with A @ f == np.cross(r, f) (model.py:25-30)."""
    x, y, z = np.asarray(r, dtype=float)
    return np.array([[0.0, -z, y],
                     [z, 0.0, -x],
                     [-y, x, 0.0]])


def _validate(positions) -> np.ndarray:
    pos = np.array(positions, dtype=float, ndmin=2)
    if pos.ndim != 2 or pos.shape[1] != 3 or pos.shape[0] < 1:
        raise ValueError(f"positions must be (n, 3) with n >= 1, got {pos.shape}")
    if not np.isfinite(pos).all():
        raise ValueError("positions must be finite")
    return pos


def _raise_dup(hit):
    body, i, j, tol = hit
    if i < 0:
        raise DuplicateBeadsError("all beads coincide")
    raise DuplicateBeadsError(f"beads {i} and {j} are closer than {tol:.3e} (dup_tol)")


class BeadModel:
    """One rigid body: an ordered (n, 3) array of distinct, finite positions
    (model.py:33-62).  Immutable after construction."""

    def __init__(self, positions, body_id: int = 0, *, check_duplicates: bool = True):
        pos = _validate(positions)
        if check_duplicates and pos.shape[0] >= 2:
            hit = _gpu_check_duplicates(pos, np.array([0, pos.shape[0]], np.int64))
            if hit is not None:
                _raise_dup(hit)
        pos.flags.writeable = False
        self.positions = pos
        self.body_id = int(body_id)

    @property
    def n(self) -> int:
        return self.positions.shape[0]

    @property
    def centroid(self) -> np.ndarray:
        c = getattr(self, "_centroid", None)
        if c is None:
            c = self._centroid = self.positions.mean(axis=0)
        return c

    def __repr__(self):
        return f"BeadModel(n={self.n}, body_id={self.body_id})"


def centroid(model: BeadModel) -> np.ndarray:
    """Arithmetic mean of the bead positions (model.py:81-83)."""
    return model.centroid.copy()


class MultiBodyModel:
    """Ordered collection of rigid bodies; fixes the global 3n vector layout
    (model.py:86-110).  ``from_arrays`` builds one from concatenated positions
    and offsets with a single batched GPU duplicate check."""

    def __init__(self, bodies):
        bodies = list(bodies)
        if not bodies:
            raise ValueError("need at least one body")
        self.bodies = bodies
        counts = np.array([b.n for b in bodies])
        self.offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        self._positions = None

    @classmethod
    def from_arrays(cls, positions, offsets, check_duplicates: bool = True):
        pos = _validate(positions)
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        if offsets.ndim != 1 or len(offsets) < 2 or offsets[0] != 0 or offsets[-1] != pos.shape[0] \
                or np.any(np.diff(offsets) < 1):
            raise ValueError("offsets must be 0 = o_0 < o_1 < ... < o_m = n_total")
        if check_duplicates:
            hit = _gpu_check_duplicates(pos, offsets)
            if hit is not None:
                _raise_dup(hit)
        pos.flags.writeable = False
        self = cls.__new__(cls)
        self.offsets = offsets
        self._positions = pos
        self.bodies = _LazyBodies(pos, offsets)
        return self

    @property
    def positions(self) -> np.ndarray:
        if self._positions is None:
            self._positions = np.concatenate([b.positions for b in self.bodies])
        return self._positions

    @property
    def m(self) -> int:
        return len(self.offsets) - 1

    @property
    def n_total(self) -> int:
        return int(self.offsets[-1])

    def __iter__(self):
        return iter(self.bodies)

    def __repr__(self):
        return f"MultiBodyModel(m={self.m}, n_total={self.n_total})"


class _LazyBodies:
    """Sequence of BeadModel views over concatenated positions (already checked)."""

    def __init__(self, pos, offsets):
        self._pos, self._off = pos, offsets

    def __len__(self):
        return len(self._off) - 1

    def __getitem__(self, j):
        if isinstance(j, slice):
            return [self[i] for i in range(*j.indices(len(self)))]
        if j < 0:
            j += len(self)
        if not 0 <= j < len(self):
            raise IndexError(j)
        return BeadModel(self._pos[self._off[j]:self._off[j + 1]], body_id=j, check_duplicates=False)

    def __iter__(self):
        return (self[j] for j in range(len(self)))


@dataclass(frozen=True)
class ZMatrix:
    """Dense 6 x 3n resultant matrix about ``origin`` (model.py:113-126).

    ``entries`` is materialized for compatibility; ``zf`` / ``ztu`` contract
    Z on the GPU without forming it.
    """

    entries: np.ndarray
    origin: np.ndarray = field(default_factory=lambda: np.zeros(3))
    positions: np.ndarray | None = None

    @property
    def n(self) -> int:
        return self.entries.shape[1] // 3

    def _plan(self):
        from ._plan import Plan

        p = getattr(self, "_p", None)
        if p is None:
            p = Plan(self.positions, np.array([0, self.positions.shape[0]], np.int64))
            object.__setattr__(self, "_p", p)
        return p

    def zf(self, f):
        """Z @ f on the GPU (f: (3n,) or (3n, k))."""
        f = np.asarray(f, dtype=float)
        single = f.ndim == 1
        f2 = np.ascontiguousarray(f.reshape(3 * self.n, -1))
        out = self._plan().z(L.Z_F, f2, origin=self.origin.reshape(1, 3))
        return out[:, 0] if single else out

    def ztu(self, u):
        """Z.T @ u on the GPU (u: (6,) or (6, k))."""
        u = np.asarray(u, dtype=float)
        single = u.ndim == 1
        u2 = np.ascontiguousarray(u.reshape(6, -1))
        out = self._plan().z(L.Z_TU, u2, origin=self.origin.reshape(1, 3))
        return out[:, 0] if single else out


def assemble_z(model: BeadModel, origin=None) -> ZMatrix:
    """Dense resultant matrix of ``model`` about ``origin`` (model.py:129-149);
    the origin defaults to the centroid."""
    origin = model.centroid if origin is None else np.asarray(origin, dtype=float)
    n = model.n
    z = np.zeros((6, 3 * n))
    z[:3] = np.tile(np.eye(3), n)
    rel = model.positions - origin
    x, y, zc = rel[:, 0], rel[:, 1], rel[:, 2]
    rot = z[3:].reshape(3, n, 3)
    rot[0, :, 1] = -zc
    rot[0, :, 2] = y
    rot[1, :, 0] = zc
    rot[1, :, 2] = -x
    rot[2, :, 0] = -y
    rot[2, :, 1] = x
    return ZMatrix(z, np.array(origin, dtype=float).copy(), model.positions)
