"""Multi-process path with the CUDA operators (the GPU pool gives one GPU per call, so the ranks
share it and talk over gloo; NCCL refuses two ranks on one device).  Every rank builds its
ShardedMultiBodyOperator shard on the GPU, applies it, and the gathered result must equal a
single-process MultiBodyOperator bitwise: per-body results do not depend on the split.  The
bench's multi-rank mode (strong sharding, max-over-ranks timing, gather) runs end to end."""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def rq():
    import paper_1708_08427_b200 as rq
    from paper_1708_08427_b200 import _lib

    if _lib.device_count() < 1:
        pytest.fail("no GPU visible: the gpu tests must run on a B200 (no CPU fallback)")
    return rq


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, pos, off, v, g, result):
    import torch
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    from paper_1708_08427_b200.parallel import ShardedMultiBodyOperator

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sh = ShardedMultiBodyOperator(pos, off, rank, world)
        outs = {}
        for name, x in (("qtilde_v", v), ("qtilde_tv", g), ("qv", v)):
            y = sh.apply_global(name, x)  # numpy in -> numpy out through the host path
            outs[name] = sh.gather(name, torch.from_numpy(np.ascontiguousarray(y))).numpy()
        if rank == 0:
            result.put({k: o.tolist() for k, o in outs.items()})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_cuda_operators_gather_bitwise(rq, world):
    import torch.multiprocessing as mp

    from paper_1708_08427_b200.workloads import ellipsoid_batch

    sizes = [4096] * 6 + [50000, 300, 3] if world == 2 else [5000, 7000]  # world 3: an empty shard
    pos, off = ellipsoid_batch(sizes, seed=21)
    rng = np.random.default_rng(4)
    N, m = int(off[-1]), len(off) - 1
    v = rng.normal(size=3 * N)
    g = rng.normal(size=3 * N - 6 * m)
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, pos, off, v, g, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get()  # before join: the result is large enough to fill the pipe
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    op = rq.MultiBodyOperator(rq.MultiBodyModel.from_arrays(pos, off))
    for name, x in (("qv", v), ("qtilde_v", v)):
        np.testing.assert_array_equal(np.array(got[name]), op.apply(name, x), err_msg=name)
    np.testing.assert_array_equal(np.array(got["qtilde_tv"]), op.apply("qtilde_tv", g))


def test_bench_two_ranks_functional(tmp_path):
    """bench.py --gpus 2 under torchrun (ranks sharing the GPU over gloo, RQ_BENCH_SHARE_GPU=1):
    strong sharding, one JSON line from rank 0 with the job's beads, the gather timed."""
    env = dict(os.environ, RQ_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "5", "--warmup", "3", "--scale", "0.05", "--no-e2e"]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = lines[0]
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert d["gather"] is not None and d["gather"]["bytes"] > 0
    assert d["config"]["sharding"].startswith("strong")


def test_bench_nccl_single_rank(tmp_path):
    """The NCCL calls of the multi-rank bench path (process group bound to the device, all_reduce,
    barrier, the max-padded all_gather of the shard outputs) on the one GPU the pool gives:
    torchrun with one rank, process group forced (RQ_BENCH_FORCE_DIST=1)."""
    env = dict(os.environ, RQ_BENCH_FORCE_DIST="1")
    env.pop("RQ_BENCH_SHARE_GPU", None)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "1", "--steps", "5", "--warmup", "3", "--scale", "0.05", "--no-e2e", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=ROOT, timeout=600)
    if r.returncode != 0 and any(m in r.stderr for m in ("ncclSystemError", "ncclUnhandledCudaError",
                                                         "ncclInternalError", "unhandled system error")):
        pytest.skip("NCCL could not initialise on this box: " + r.stderr[-300:])
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = lines[0]
    assert d["n_gpus"] == 1 and d["value"] > 0
    assert d["gather"] is not None and d["gather"]["bytes"] > 0 and d["gather"]["ms"] > 0
