"""Owning handle around an rq_plan (device-resident tree + factors + apply
layout for a batch of bodies) and the vector plumbing of the C ABI.

Vectors may be numpy arrays (copied host->device->host inside the library,
``rq_apply_host``) or contiguous float64 CUDA torch tensors (zero-copy,
``rq_apply`` on torch's current stream).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L


def _is_torch_cuda(x) -> bool:
    return type(x).__module__.startswith("torch") and getattr(x, "is_cuda", False)


def host_result(shape):
    """A float64 result array for the host path, in page-locked memory when torch can give it
    (its caching host allocator reuses freed blocks), so the device-to-host copy lands directly
    in the returned array instead of going through a staging buffer and a second memcpy.
    RQ_PINNED_RESULTS=0 returns plain numpy memory."""
    import os

    if os.environ.get("RQ_PINNED_RESULTS", "1") != "0":
        try:
            import torch

            if torch.cuda.is_available():
                return torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()
        except (ImportError, RuntimeError):
            pass
    return np.empty(shape)


def _torch_stream(device=None):
    import torch

    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


class Plan:
    def __init__(self, positions, offsets, max_depth: int = 96, check_duplicates: bool = False):
        lib = L.lib()
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        self.m = len(offsets) - 1
        self.offsets = offsets
        flags = L.SETUP_CHECK_DUPS if check_duplicates else 0
        stream = None
        if _is_torch_cuda(positions):
            pos = positions.contiguous()
            import torch

            if pos.dtype != torch.float64:
                pos = pos.double()
            stream = _torch_stream()
            self._keep = pos
        else:
            pos = np.ascontiguousarray(positions, dtype=float).reshape(-1, 3)
            flags |= L.SETUP_HOST_INPUT
            self._keep = pos
        h = C.c_void_p()
        L.check(lib.rq_setup(L.ptr(pos), offsets.ctypes.data_as(C.POINTER(C.c_int64)), self.m, int(max_depth),
                             flags, stream, C.byref(h)))
        self._h = h
        self._keep = None
        self.n = np.diff(offsets)
        self.N = int(offsets[-1])

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                L.lib().rq_plan_free(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    def info(self) -> dict:
        inf = L.PlanInfo()
        L.check(L.lib().rq_plan_get_info(self._h, C.byref(inf)))
        d = {k: getattr(inf, k) for k, _ in L.PlanInfo._fields_
             if k not in ("n_case", "sweep_bytes", "mrhs_units", "mrhs_bytes")}
        d["sweep_bytes"] = {"up": inf.sweep_bytes[0], "down": inf.sweep_bytes[1]}
        d["mrhs_units"] = {"tiles": inf.mrhs_units[0], "tops": inf.mrhs_units[1]}
        d["mrhs_bytes"] = {"tiles": inf.mrhs_bytes[0], "tops": inf.mrhs_bytes[1]}
        d["n_case"] = list(inf.n_case)
        return d

    def release_stream(self, stream):
        """Free the exchange state this plan keeps for a CUDA stream (torch.cuda.Stream or raw
        handle) after synchronising it; rq_plan_release_stream."""
        h = getattr(stream, "cuda_stream", stream)
        L.check(L.lib().rq_plan_release_stream(self._h, C.c_void_p(h)))

    def _check_device(self, t):
        dev = L.lib().rq_plan_device(self._h)
        if t.device.index != dev:
            raise ValueError(f"tensor on cuda:{t.device.index}, operator on cuda:{dev}")

    # ---- lengths -------------------------------------------------------------
    def lengths(self, op: str):
        full = 3 * self.N
        comp = 3 * self.N - 6 * self.m
        return {"qv": (full, full), "qtv": (full, full), "qtilde_v": (full, comp),
                "qtilde_tv": (comp, full)}[op]

    # ---- application -----------------------------------------------------------
    def apply(self, op: str, v2):
        """v2: (in_len, k) C-contiguous float64 numpy array or CUDA tensor."""
        code = L.OPS[op]
        li, lo = self.lengths(op)
        k = int(v2.shape[1])
        lib = L.lib()
        if _is_torch_cuda(v2):
            import torch

            out = torch.empty((lo, k), dtype=torch.float64, device=v2.device)
            self._check_device(v2)
            L.check(lib.rq_apply(self._h, code, v2.data_ptr(), out.data_ptr(), k, _torch_stream(v2.device)))
            return out
        out = host_result((lo, k))
        L.check(lib.rq_apply_host(self._h, code, v2.ctypes.data, out.ctypes.data, k))
        return out

    def apply_host_many(self, items):
        """[(op, (in_len, k) numpy array), ...] -> results, every application queued on the
        host-async path (rq_apply_host_async) before one rq_host_wait, so the H2D of one
        operand overlaps the D2H of the previous result."""
        lib = L.lib()
        outs = []
        try:
            for op, v2 in items:
                _, lo = self.lengths(op)
                k = int(v2.shape[1])
                out = host_result((lo, k))
                outs.append((out, v2))  # both stay referenced until the wait
                L.check(lib.rq_apply_host_async(self._h, L.OPS[op], v2.ctypes.data, out.ctypes.data, k))
        finally:
            L.check(lib.rq_host_wait(self._h))
        return [o for o, _ in outs]

    def z(self, op: int, v2, origin=None):
        lib = L.lib()
        k = int(v2.shape[1])
        lo = 6 * self.m if op == L.Z_F else 3 * self.N
        org = None
        if origin is not None:
            org = np.ascontiguousarray(origin, dtype=float).reshape(self.m, 3)
        optr = org.ctypes.data if org is not None else None
        if _is_torch_cuda(v2):
            import torch

            out = torch.empty((lo, k), dtype=torch.float64, device=v2.device)
            self._check_device(v2)
            L.check(lib.rq_z_apply(self._h, op, v2.data_ptr(), out.data_ptr(), k, optr, _torch_stream(v2.device)))
            return out
        out = host_result((lo, k))
        L.check(lib.rq_z_apply_host(self._h, op, v2.ctypes.data, out.ctypes.data, k, optr))
        return out

    def centroids(self) -> np.ndarray:
        out = np.empty((self.m, 3))
        L.check(L.lib().rq_body_centroids(self._h, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    # ---- parity exports -------------------------------------------------------------
    def export_tree(self, body: int = 0) -> dict:
        n = int(self.n[body])
        nn = 2 * n - 1
        i64 = lambda c: np.empty(c, np.int64)  # noqa: E731
        d = dict(perm=i64(n), start=i64(nn), stop=i64(nn), left=i64(nn), right=i64(nn),
                 split_axis=np.empty(nn, np.int32), depth=np.empty(nn, np.int32),
                 centroid=np.empty((nn, 3)), box=np.empty((nn, 2, 3)))
        P = lambda a, t: a.ctypes.data_as(C.POINTER(t))  # noqa: E731
        L.check(L.lib().rq_export_tree(self._h, body, P(d["perm"], C.c_int64), P(d["start"], C.c_int64),
                                       P(d["stop"], C.c_int64), P(d["left"], C.c_int64),
                                       P(d["right"], C.c_int64), P(d["split_axis"], C.c_int32),
                                       P(d["depth"], C.c_int32), P(d["centroid"], C.c_double),
                                       P(d["box"], C.c_double)))
        return d

    def export_factors(self, body: int = 0, omega: bool = True) -> dict:
        n = int(self.n[body])
        nn = 2 * n - 1
        lib = L.lib()
        d = dict(case=np.empty(nn, np.int32), n=np.empty(nn, np.int64), nx=np.empty(nn, np.int64),
                 ny=np.empty(nn, np.int64), swapped=np.empty(nn, np.uint8), t22=np.empty((nn, 3, 3)),
                 res_offsets=np.empty(nn, np.int64), total_rows=np.empty(1, np.int64))
        om = None
        if omega:
            sz = lib.rq_omega_size(self._h, body)
            if sz < 0:
                L.check(7)
            om = np.empty(max(int(sz), 1))
        P = lambda a, t: a.ctypes.data_as(C.POINTER(t))  # noqa: E731
        L.check(lib.rq_export_factors(self._h, body, P(d["case"], C.c_int32), P(d["n"], C.c_int64),
                                      P(d["nx"], C.c_int64), P(d["ny"], C.c_int64), P(d["swapped"], C.c_uint8),
                                      P(d["t22"], C.c_double), P(om, C.c_double) if om is not None else None,
                                      P(d["res_offsets"], C.c_int64), P(d["total_rows"], C.c_int64)))
        d["omega_flat"] = om
        d["total_rows"] = int(d["total_rows"][0])
        return d

    def explicit_q(self, body: int = 0):
        lib = L.lib()
        nb = np.zeros(1, np.int64)
        nd = np.zeros(1, np.int64)
        P = lambda a, t: a.ctypes.data_as(C.POINTER(t))  # noqa: E731
        L.check(lib.rq_explicit_q_size(self._h, body, P(nb, C.c_int64), P(nd, C.c_int64)))
        n = int(self.n[body])
        root = np.empty((6, 3 * n))
        bnode = np.empty(max(int(nb[0]), 1), np.int64)
        bcol = np.empty_like(bnode)
        brows = np.empty_like(bnode)
        data = np.empty(max(int(nd[0]), 1))
        L.check(lib.rq_explicit_q(self._h, body, P(root, C.c_double), P(bnode, C.c_int64), P(bcol, C.c_int64),
                                  P(brows, C.c_int64), P(data, C.c_double)))
        tr = self.export_tree(body)
        out = []
        off = 0
        for b in range(int(nb[0])):
            node, col, rows = int(bnode[b]), int(bcol[b]), int(brows[b])
            width = 3 * int(tr["stop"][node] - tr["start"][node])  # a block spans its node's beads
            out.append((node, col, data[off:off + rows * width].reshape(rows, width).copy()))
            off += rows * width
        return root, out


def check_duplicates(positions, offsets):
    """GPU duplicate-bead check (model.py:65-78); returns None or (body, i, j, tol)."""
    pos = np.ascontiguousarray(positions, dtype=float).reshape(-1, 3)
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    b = np.zeros(1, np.int64)
    i = np.zeros(1, np.int64)
    j = np.zeros(1, np.int64)
    t = np.zeros(1)
    P = lambda a, tt: a.ctypes.data_as(C.POINTER(tt))  # noqa: E731
    rc = L.lib().rq_check_duplicates(pos.ctypes.data, P(offsets, C.c_int64), len(offsets) - 1,
                                     L.SETUP_HOST_INPUT, None, P(b, C.c_int64), P(i, C.c_int64),
                                     P(j, C.c_int64), P(t, C.c_double))
    if rc == L.RQ_OK:
        return None
    if rc != 1:
        L.check(rc)
    return int(b[0]), int(i[0]), int(j[0]), float(t[0])
