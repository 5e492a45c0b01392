"""ctypes binding of librigidq_b200.so (include/rigidq_b200.h).

The product path has no CPU fallback: if the shared library is missing this
module raises on first use, and every entry point that needs a GPU raises
RuntimeError when none is visible.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from . import errors as E

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RQ_LIB_PATH") or os.path.join(HERE, "librigidq_b200.so")

OP_QV, OP_QTV, OP_QTILDE_V, OP_QTILDE_TV = 0, 1, 2, 3
OPS = {"qv": OP_QV, "qtv": OP_QTV, "qtilde_v": OP_QTILDE_V, "qtilde_tv": OP_QTILDE_TV}
Z_F, Z_TU = 0, 1
SETUP_HOST_INPUT, SETUP_CHECK_DUPS = 1, 2

RQ_OK = 0
_ERRS = {
    1: E.DuplicateBeadsError,
    2: ValueError,
    3: E.BodyTooSmallError,
    4: E.LengthMismatchError,
    5: E.TooSmallError,
    6: E.SizeGuardError,
    7: RuntimeError,
    8: MemoryError,
}

# (name, restype, argtypes) for every symbol of include/rigidq_b200.h
_dp, _ip, _i32p, _u8p, _vp = (C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_int32),
                              C.POINTER(C.c_uint8), C.c_void_p)


class PlanInfo(C.Structure):
    _fields_ = [("m", C.c_int64), ("n_beads", C.c_int64), ("n_nodes", C.c_int64), ("n_streams", C.c_int64),
                ("n_steps", C.c_int64), ("n_top", C.c_int64), ("tile_leaves", C.c_int64), ("n_tiles", C.c_int64),
                ("blob_bytes", C.c_int64), ("sweep_bytes", C.c_int64 * 2), ("record_doubles", C.c_int64),
                ("full_len", C.c_int64), ("comp_len", C.c_int64), ("n_case", C.c_int64 * 4),
                ("device_bytes", C.c_int64), ("rounds", C.c_int64),
                ("node_slots", C.c_int64), ("stage_bytes", C.c_int64), ("sweep_smem", C.c_int64),
                ("sweep_ctas_per_sm", C.c_int64), ("top_staged", C.c_int64), ("top_global", C.c_int64),
                ("mrhs_min_k", C.c_int64), ("mrhs_units", C.c_int64 * 2), ("mrhs_bytes", C.c_int64 * 2)]


SIGNATURES = [
    ("rq_last_error", C.c_char_p, []),
    ("rq_device_count", C.c_int, []),
    ("rq_version", C.c_int, []),
    ("rq_setup", C.c_int, [_vp, _ip, C.c_int64, C.c_int, C.c_uint32, _vp, C.POINTER(_vp)]),
    ("rq_plan_free", C.c_int, [_vp]),
    ("rq_plan_get_info", C.c_int, [_vp, C.POINTER(PlanInfo)]),
    ("rq_plan_device", C.c_int, [_vp]),
    ("rq_plan_release_stream", C.c_int, [_vp, _vp]),
    ("rq_apply", C.c_int, [_vp, C.c_int, _vp, _vp, C.c_int64, _vp]),
    ("rq_apply_ex", C.c_int, [_vp, C.c_int, _vp, _vp, C.c_int64, _vp, C.c_uint32]),
    ("rq_launches_per_apply", C.c_int, [_vp, C.c_int, C.c_int64]),
    ("rq_apply_host", C.c_int, [_vp, C.c_int, _vp, _vp, C.c_int64]),
    ("rq_apply_host_async", C.c_int, [_vp, C.c_int, _vp, _vp, C.c_int64]),
    ("rq_host_wait", C.c_int, [_vp]),
    ("rq_z_apply", C.c_int, [_vp, C.c_int, _vp, _vp, C.c_int64, _vp, _vp]),
    ("rq_z_apply_host", C.c_int, [_vp, C.c_int, _vp, _vp, C.c_int64, _vp]),
    ("rq_body_centroids", C.c_int, [_vp, _dp]),
    ("rq_check_duplicates", C.c_int, [_vp, _ip, C.c_int64, C.c_uint32, _vp, _ip, _ip, _ip, _dp]),
    ("rq_export_tree", C.c_int, [_vp, C.c_int64, _ip, _ip, _ip, _ip, _ip, _i32p, _i32p, _dp, _dp]),
    ("rq_export_factors", C.c_int, [_vp, C.c_int64, _i32p, _ip, _ip, _ip, _u8p, _dp, _dp, _ip, _ip]),
    ("rq_omega_size", C.c_int64, [_vp, C.c_int64]),
    ("rq_explicit_q_size", C.c_int, [_vp, C.c_int64, _ip, _ip]),
    ("rq_explicit_q", C.c_int, [_vp, C.c_int64, _dp, _ip, _ip, _ip, _dp]),
    ("rq_small_lq", C.c_int, [_dp, C.c_int, C.c_int64, _dp, _dp]),
    ("rq_factor_bead_bead", C.c_int, [_dp, C.c_int64, _dp, _dp]),
    ("rq_node_merge", C.c_int, [C.c_int, _dp, C.c_double, C.c_double, _dp, _dp, C.c_int64, _dp, _dp]),
    ("rq_node_split", C.c_int, [C.c_int, _dp, C.c_double, C.c_double, _dp, _dp, C.c_int64, _dp, _dp]),
]

_lib = None
_lock = threading.Lock()


def lib():
    """Load the CUDA library (fails loudly when it was not built)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(
                        f"{LIB_PATH} is missing: the B200 CUDA library has not been built "
                        "(run `python -c 'import __graft_entry__ as g; g.build()'`); there is no CPU fallback")
                L = C.CDLL(LIB_PATH)
                for name, res, args in SIGNATURES:
                    fn = getattr(L, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = L
    return _lib


def check(rc: int):
    if rc != RQ_OK:
        msg = lib().rq_last_error().decode(errors="replace")
        raise _ERRS.get(rc, RuntimeError)(msg)


def device_count() -> int:
    return int(lib().rq_device_count())


def ptr(a) -> int:
    """Raw address of a numpy array or a torch tensor."""
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data
