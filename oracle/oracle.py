"""ctypes front end of the C oracle (rq_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg -- never by the product
package.  The oracle restates /root/reference/pkg/src/rigidq (tree.py,
factor.py, matfree.py, model.py) in C; it is pinned against the reference
through tests/golden/ (see tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "librq_oracle.so")

LEAF, BEAD_BEAD, RIGID_BEAD, GENERAL = 0, 1, 2, 3
OPS = {"qv": 0, "qtv": 1, "qtilde_v": 2, "qtilde_tv": 3}


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


class _Body(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("nn", C.c_int64), ("root", C.c_int64),
        ("perm", C.POINTER(C.c_int64)), ("pos", C.POINTER(C.c_double)),
        ("start", C.POINTER(C.c_int64)), ("stop", C.POINTER(C.c_int64)),
        ("left", C.POINTER(C.c_int64)), ("right", C.POINTER(C.c_int64)),
        ("split_axis", C.POINTER(C.c_int32)), ("depth", C.POINTER(C.c_int32)),
        ("centroid", C.POINTER(C.c_double)), ("box", C.POINTER(C.c_double)),
        ("fcase", C.POINTER(C.c_int32)), ("fn", C.POINTER(C.c_int64)),
        ("fnx", C.POINTER(C.c_int64)), ("fny", C.POINTER(C.c_int64)),
        ("swapped", C.POINTER(C.c_uint8)), ("t22", C.POINTER(C.c_double)),
        ("omega_off", C.POINTER(C.c_int64)), ("omega_k", C.POINTER(C.c_int32)),
        ("omega", C.POINTER(C.c_double)), ("res_offsets", C.POINTER(C.c_int64)),
        ("total_rows", C.c_int64),
    ]


class _Batch(C.Structure):
    _fields_ = [("m", C.c_int64), ("offsets", C.POINTER(C.c_int64)),
                ("bodies", C.POINTER(_Body))]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int64)
        L.rqo_body_setup.argtypes = [dp, C.c_int64, C.c_int, C.POINTER(_Body)]
        L.rqo_body_free.argtypes = [C.POINTER(_Body)]
        L.rqo_upward.argtypes = [C.POINTER(_Body), dp, dp, C.c_int64]
        L.rqo_downward.argtypes = [C.POINTER(_Body), dp, dp, C.c_int64]
        L.rqo_small_lq.argtypes = [dp, C.c_int, dp, dp]
        L.rqo_check_duplicates.argtypes = [dp, C.c_int64, ip, ip]
        L.rqo_batch_setup.argtypes = [dp, ip, C.c_int64, C.c_int, C.c_int, C.POINTER(_Batch)]
        L.rqo_batch_free.argtypes = [C.POINTER(_Batch)]
        L.rqo_batch_apply.argtypes = [C.POINTER(_Batch), C.c_int, dp, dp, C.c_int64, C.c_int]
        L.rqo_batch_zf.argtypes = [dp, ip, C.c_int64, dp, dp, C.c_int]
        L.rqo_batch_ztu.argtypes = [dp, ip, C.c_int64, dp, dp, C.c_int]
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int64))


def _arr(ptr, count, dtype):
    if count == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(count,)).astype(dtype, copy=True)


class DuplicateBeads(Exception):
    pass


def small_lq(a):
    a = np.ascontiguousarray(a, dtype=float)
    k = a.shape[1]
    t = np.zeros((3, 3))
    om = np.zeros((k, k))
    lib().rqo_small_lq(_dp(a), k, _dp(t), _dp(om))
    return t, om


def check_duplicates(pos):
    pos = np.ascontiguousarray(pos, dtype=float)
    i = np.zeros(1, np.int64)
    j = np.zeros(1, np.int64)
    found = lib().rqo_check_duplicates(_dp(pos), pos.shape[0], _ip(i), _ip(j))
    return (int(i[0]), int(j[0])) if found else None


class OracleBody:
    """Tree + factor table of one body (reference BodyOperator, matfree.py:173-206)."""

    def __init__(self, positions, max_depth: int = 96):
        pos = np.ascontiguousarray(positions, dtype=float).reshape(-1, 3)
        self._b = _Body()
        rc = lib().rqo_body_setup(_dp(pos), pos.shape[0], max_depth, C.byref(self._b))
        if rc == 1:
            raise DuplicateBeads("split depth exceeded (near-coincident beads)")
        if rc != 0:
            raise RuntimeError(f"oracle setup failed rc={rc}")
        b = self._b
        n, nn = b.n, b.nn
        self.n = n
        self.root_id = b.root
        self.perm = _arr(b.perm, n, np.int64)
        self.positions = _arr(b.pos, 3 * n, float).reshape(n, 3)
        self.start = _arr(b.start, nn, np.int64)
        self.stop = _arr(b.stop, nn, np.int64)
        self.left = _arr(b.left, nn, np.int64)
        self.right = _arr(b.right, nn, np.int64)
        self.split_axis = _arr(b.split_axis, nn, np.int32)
        self.depth = _arr(b.depth, nn, np.int32)
        self.centroid = _arr(b.centroid, 3 * nn, float).reshape(nn, 3)
        self.box = _arr(b.box, 6 * nn, float).reshape(nn, 2, 3)
        self.case = _arr(b.fcase, nn, np.int32)
        self.fn = _arr(b.fn, nn, np.int64)
        self.fnx = _arr(b.fnx, nn, np.int64)
        self.fny = _arr(b.fny, nn, np.int64)
        self.swapped = _arr(b.swapped, nn, np.uint8).astype(bool)
        self.t22 = _arr(b.t22, 9 * nn, float).reshape(nn, 3, 3)
        off = _arr(b.omega_off, nn, np.int64)
        ks = _arr(b.omega_k, nn, np.int32)
        tot = int(sum(int(k) * int(k) for k in ks))
        flat = _arr(b.omega, tot, float)
        self.omega = [None if ks[i] == 0 else flat[off[i]:off[i] + ks[i] * ks[i]].reshape(ks[i], ks[i])
                      for i in range(nn)]
        self.res_offsets = _arr(b.res_offsets, nn, np.int64)
        self.total_rows = int(b.total_rows)

    def __del__(self):
        try:
            lib().rqo_body_free(C.byref(self._b))
        except Exception:
            pass

    def _cols(self, v, length):
        v = np.asarray(v, dtype=float)
        single = v.ndim == 1
        v2 = np.ascontiguousarray(v.reshape(length, -1))
        return v2, single

    def qv(self, v):
        v2, single = self._cols(v, 3 * self.n)
        out = np.zeros_like(v2)
        lib().rqo_upward(C.byref(self._b), _dp(v2), _dp(out), v2.shape[1])
        return out[:, 0] if single else out

    def qtv(self, w):
        w2, single = self._cols(w, 3 * self.n)
        out = np.zeros_like(w2)
        lib().rqo_downward(C.byref(self._b), _dp(w2), _dp(out), w2.shape[1])
        return out[:, 0] if single else out

    def qtilde_v(self, v):
        return self.qv(v)[6:]

    def qtilde_tv(self, g):
        g = np.asarray(g, dtype=float)
        single = g.ndim == 1
        g2 = g.reshape(3 * self.n - 6, -1)
        w = np.zeros((3 * self.n, g2.shape[1]))
        w[6:] = g2
        out = self.qtv(w)
        return out[:, 0] if single else out


class OracleBatch:
    """Multi-body oracle with OpenMP over bodies (MultiBodyOperator, matfree.py:212-247)."""

    def __init__(self, positions, offsets, max_depth: int = 96, threads: int | None = None):
        self.pos = np.ascontiguousarray(positions, dtype=float).reshape(-1, 3)
        self.offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        self.m = len(self.offsets) - 1
        self.threads = threads or os.cpu_count() or 1
        self._b = _Batch()
        rc = lib().rqo_batch_setup(_dp(self.pos), _ip(self.offsets), self.m, max_depth,
                                   self.threads, C.byref(self._b))
        if rc != 0:
            raise DuplicateBeads("oracle batch setup failed")

    def __del__(self):
        try:
            lib().rqo_batch_free(C.byref(self._b))
        except Exception:
            pass

    def lengths(self, op):
        n = np.diff(self.offsets)
        full = int(3 * n.sum())
        comp = int(3 * n.sum() - 6 * self.m)
        return {"qv": (full, full), "qtv": (full, full),
                "qtilde_v": (full, comp), "qtilde_tv": (comp, full)}[op]

    def apply(self, op, v):
        li, lo = self.lengths(op)
        v = np.asarray(v, dtype=float)
        single = v.ndim == 1
        v2 = np.ascontiguousarray(v.reshape(li, -1))
        out = np.zeros((lo, v2.shape[1]))
        rc = lib().rqo_batch_apply(C.byref(self._b), OPS[op], _dp(v2), _dp(out), v2.shape[1], self.threads)
        if rc != 0:
            raise ValueError("body too small")
        return out[:, 0] if single else out

    def zf(self, f):
        f = np.ascontiguousarray(f, dtype=float)
        out = np.zeros(6 * self.m)
        lib().rqo_batch_zf(_dp(self.pos), _ip(self.offsets), self.m, _dp(f), _dp(out), self.threads)
        return out

    def ztu(self, u):
        u = np.ascontiguousarray(u, dtype=float)
        out = np.zeros(3 * self.pos.shape[0])
        lib().rqo_batch_ztu(_dp(self.pos), _ip(self.offsets), self.m, _dp(u), _dp(out), self.threads)
        return out
