"""Host-buffer applications (rq_apply_host / rq_apply_host_async + rq_host_wait).

Pinned and pageable host buffers, synchronous and queued back to back (two
staging slots: the H2D of one application overlaps the D2H of the previous
one; a third queued application completes the first).  Every result must
equal the device-resident application bitwise: same kernels, same data.
"""

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


def _device(op, name, x):
    import torch

    return op.apply(name, torch.from_numpy(x).cuda()).cpu().numpy()


@pytest.mark.parametrize("counts", [[4096] * 60, [3000, 60000, 700, 90000, 2500, 40000], [50, 3, 2000, 7, 4096, 300]])
def test_host_paths_equal_device(rq, counts):
    import torch
    from paper_1708_08427_b200 import _lib as L
    from paper_1708_08427_b200.workloads import ellipsoid_batch

    pos, off = ellipsoid_batch(counts, seed=11)
    op = rq.MultiBodyOperator(rq.MultiBodyModel.from_arrays(pos, off))
    N, m = int(off[-1]), len(off) - 1
    lib, h = L.lib(), op.plan.handle
    rng = np.random.default_rng(5)
    vs = [rng.normal(size=3 * N) for _ in range(3)]
    gs = [rng.normal(size=3 * N - 6 * m) for _ in range(3)]
    want_v = [_device(op, "qtilde_v", v) for v in vs]
    want_g = [_device(op, "qtilde_tv", g) for g in gs]
    for pinned in (True, False):
        def buf(x):
            t = torch.from_numpy(np.array(x))
            return t.pin_memory() if pinned else t
        hv = [buf(v) for v in vs]
        hg = [buf(g) for g in gs]
        ov = [buf(np.full(3 * N - 6 * m, np.nan)) for _ in vs]
        og = [buf(np.full(3 * N, np.nan)) for _ in gs]
        # synchronous
        L.check(lib.rq_apply_host(h, L.OP_QTILDE_V, hv[0].data_ptr(), ov[0].data_ptr(), 1))
        assert np.array_equal(ov[0].numpy(), want_v[0]), pinned
        # queued back to back: six applications, two slots (each new one completes an older one)
        for i in range(3):
            L.check(lib.rq_apply_host_async(h, L.OP_QTILDE_V, hv[i].data_ptr(), ov[i].data_ptr(), 1))
            L.check(lib.rq_apply_host_async(h, L.OP_QTILDE_TV, hg[i].data_ptr(), og[i].data_ptr(), 1))
        L.check(lib.rq_host_wait(h))
        for i in range(3):
            assert np.array_equal(ov[i].numpy(), want_v[i]), (pinned, i)
            assert np.array_equal(og[i].numpy(), want_g[i]), (pinned, i)


def test_numpy_api_and_full_ops_equal_device(rq):
    from paper_1708_08427_b200.workloads import ellipsoid_batch

    pos, off = ellipsoid_batch([4096] * 40 + [1, 2, 777], seed=12)
    op = rq.MultiBodyOperator(rq.MultiBodyModel.from_arrays(pos, off))
    N = int(off[-1])
    rng = np.random.default_rng(6)
    v = rng.normal(size=3 * N)
    for name in ("qv", "qtv"):
        assert np.array_equal(op.apply(name, v), _device(op, name, v)), name
    V = rng.normal(size=(3 * N, 3))
    assert np.array_equal(op.apply("qv", V), op.apply("qv", __import__("torch").from_numpy(V).cuda()).cpu().numpy())


def test_apply_many_and_pinned_results(rq, monkeypatch):
    """apply_many queues several host applications before one wait; its results equal
    sequential apply calls bitwise, and results live in page-locked memory by default (plain
    numpy with RQ_PINNED_RESULTS=0) -- ordinary writeable float64 arrays either way."""
    import torch

    from paper_1708_08427_b200.workloads import ellipsoid_batch

    pos, off = ellipsoid_batch([4096] * 30 + [20000, 3], seed=17)
    op = rq.MultiBodyOperator(rq.MultiBodyModel.from_arrays(pos, off))
    N, m = int(off[-1]), len(off) - 1
    rng = np.random.default_rng(8)
    vs = [rng.normal(size=3 * N) for _ in range(3)]
    gs = [rng.normal(size=3 * N - 6 * m) for _ in range(3)]
    items = [x for v, g in zip(vs, gs) for x in (("qtilde_v", v), ("qtilde_tv", g))]
    items.append(("qv", rng.normal(size=(3 * N, 2))))
    seq = [op.apply(name, x) for name, x in items]
    many = op.apply_many(items)
    for a, b in zip(many, seq):
        assert a.dtype == np.float64 and a.flags.writeable and np.array_equal(a, b)
    assert np.array_equal(seq[0], _device(op, "qtilde_v", vs[0]))
    assert torch.from_numpy(many[0]).is_pinned(), "host results should be page-locked"
    monkeypatch.setenv("RQ_PINNED_RESULTS", "0")
    plain = op.apply("qtilde_v", vs[0])
    assert not torch.from_numpy(plain).is_pinned() and np.array_equal(plain, seq[0])
