"""Host-buffer applications (rq_apply_host, the drop-in numpy path's C entry).

Pinned host buffers take the segment-pipelined path (input copies flagged per
host segment, outputs copied back per segment while the sweep runs, top-tree
residues compacted and scattered by host threads); pageable buffers take the
plain copy-apply-copy path.  Both must equal the device-resident application
bitwise: they run the same kernels on the same data.
"""

import ctypes as C

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


def _operator(rq, monkeypatch, counts, seed, rounds, segs):
    from paper_1708_08427_b200.workloads import ellipsoid_batch

    monkeypatch.setenv("RQ_WAVE_ROUNDS", str(rounds))
    monkeypatch.setenv("RQ_WAVE_SEGS", str(segs))
    pos, off = ellipsoid_batch(counts, seed=seed)
    return rq.MultiBodyOperator(rq.MultiBodyModel.from_arrays(pos, off)), off


def _device(op, name, x):
    import torch

    return op.apply(name, torch.from_numpy(x).cuda()).cpu().numpy()


@pytest.mark.parametrize("counts,rounds,segs", [
    ([4096] * 120, 16, 8),                        # many bodies, segments of whole bodies
    ([3000, 60000, 700, 90000, 2500, 40000], 12, 6),  # big bodies straddle segments; dataflow tops
    ([50, 3, 2000, 7, 4096, 300], 4, 4),          # tiny bodies, bodies without tiles
])
def test_pinned_pipelined_equals_device(rq, monkeypatch, counts, rounds, segs):
    import torch
    from paper_1708_08427_b200 import _lib as L

    op, off = _operator(rq, monkeypatch, counts, 11, rounds, segs)
    N, m = int(off[-1]), len(off) - 1
    lib = L.lib()
    h = op.plan.handle
    rng = np.random.default_rng(5)
    for rep in range(3):  # flags and counters are monotone across calls
        v = rng.normal(size=3 * N)
        g = rng.normal(size=3 * N - 6 * m)
        hv = torch.from_numpy(v).pin_memory()
        hg = torch.from_numpy(g).pin_memory()
        o1 = torch.full((3 * N - 6 * m,), np.nan, dtype=torch.float64).pin_memory()
        o2 = torch.full((3 * N,), np.nan, dtype=torch.float64).pin_memory()
        L.check(lib.rq_apply_host(h, L.OP_QTILDE_V, hv.data_ptr(), o1.data_ptr(), 1))
        L.check(lib.rq_apply_host(h, L.OP_QTILDE_TV, hg.data_ptr(), o2.data_ptr(), 1))
        assert np.array_equal(o1.numpy(), _device(op, "qtilde_v", v)), rep
        assert np.array_equal(o2.numpy(), _device(op, "qtilde_tv", g)), rep


def test_pageable_and_full_ops_equal_device(rq, monkeypatch):
    op, off = _operator(rq, monkeypatch, [4096] * 40 + [1, 2, 777], 12, 8, 4)
    N = int(off[-1])
    rng = np.random.default_rng(6)
    v = rng.normal(size=3 * N)
    for name in ("qv", "qtv"):
        assert np.array_equal(op.apply(name, v), _device(op, name, v)), name
