"""Multi-process (world_size 2, gloo, CPU) coverage of the body sharding and
the result gather (the only collective of the multi-GPU path)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1708_08427_b200.parallel import gather_shards, shard_bounds, shard_of, vector_slice


def test_shard_bounds_balanced():
    rng = np.random.default_rng(0)
    counts = np.floor(np.exp(rng.uniform(np.log(500), np.log(50000), size=2000))).astype(np.int64)
    off = np.concatenate([[0], np.cumsum(counts)])
    for world in (1, 2, 4, 8):
        b = shard_bounds(off, world)
        assert b[0] == 0 and b[-1] == len(counts) and np.all(np.diff(b) >= 0)
        beads = np.diff(off[b])
        assert beads.sum() == off[-1]
        # imbalance bounded by one body
        assert np.abs(beads - off[-1] / world).max() <= counts.max()


def test_shard_bounds_edge_cases():
    off = np.array([0, 5])
    assert list(shard_bounds(off, 1)) == [0, 1]
    b = shard_bounds(off, 3)  # more ranks than bodies: empty shards allowed
    assert b[0] == 0 and b[-1] == 1 and np.all(np.diff(b) >= 0)
    with pytest.raises(ValueError):
        shard_bounds(off, 0)


def test_vector_slices_tile_global_layout():
    off = np.array([0, 3, 10, 11, 20])
    b = shard_bounds(off, 2)
    for kind, total in (("full", 60), ("comp", 60 - 24), ("body6", 24)):
        spans = [vector_slice(off, b, r, kind) for r in range(2)]
        assert spans[0][0] == 0 and spans[-1][1] == total and spans[0][1] == spans[1][0]
    pos = np.arange(60.0).reshape(20, 3)
    p0, o0, (j0, j1) = shard_of(pos, off, 0, 2)
    p1, o1, (k0, k1) = shard_of(pos, off, 1, 2)
    assert j1 == k0 and o0[0] == 0 and o1[0] == 0
    np.testing.assert_array_equal(np.concatenate([p0, p1]), pos)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, off, result):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        b = shard_bounds(off, world)
        a, e = vector_slice(off, b, rank, "comp")
        # stand-in for the rank's operator output: a block-diagonal per-body map
        glob = torch.arange(3 * int(off[-1]) - 6 * (len(off) - 1), dtype=torch.float64)
        local = (glob[a:e] * 2.0 + rank * 0).reshape(-1, 1)
        rows = [vector_slice(off, b, r, "comp") for r in range(world)]
        out = gather_shards(local, [q - p for p, q in rows])
        if rank == 0:
            result.put(out[:, 0].numpy().tolist())
    finally:
        dist.destroy_process_group()


def test_gather_world2_gloo():
    off = np.array([0, 7, 12, 30, 31, 50, 52])
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, off, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    got = np.array(q.get())
    want = np.arange(3 * 52 - 6 * 6, dtype=float) * 2.0
    np.testing.assert_array_equal(got, want)


def test_bench_strong_sharding_covers_the_model():
    """bench.py --sharding strong: the ranks' shards concatenate to the one config-4 model."""
    import bench
    from paper_1708_08427_b200.workloads import make_config

    pos, off = make_config(4, seed=1000, scale=0.005)
    for world in (2, 3, 8):
        parts = [bench.workload(4, r, 0.005, world, True) for r in range(world)]
        assert np.array_equal(np.concatenate([p[0] for p in parts]), pos)
        sizes = np.concatenate([np.diff(p[1]) for p in parts])
        assert np.array_equal(sizes, np.diff(off))
        beads = [int(p[1][-1]) for p in parts]
        # each cut lies within half a body of its ideal position: shard sizes differ by <= 2 bodies
        assert max(beads) - min(beads) <= 2 * int(np.diff(off).max())


def _oracle_worker(rank, world, port, pos, off, v, result):
    """Each rank applies Q~ to its shard with the CPU oracle (the checker standing in for the
    CUDA operator, which needs a GPU) and the shards are gathered: the sharding + gather path
    with real operator outputs."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import OracleBatch

        b = shard_bounds(off, world)
        p_loc, o_loc, (j0, j1) = shard_of(pos, off, rank, world)
        a, e = vector_slice(off, b, rank, "full")
        if j1 > j0:
            y = OracleBatch(p_loc, o_loc, threads=1).apply("qtilde_v", v[a:e])
        else:
            y = np.zeros(0)
        rows = [vector_slice(off, b, r, "comp") for r in range(world)]
        out = gather_shards(torch.from_numpy(np.ascontiguousarray(y)), [q - p for p, q in rows])
        if rank == 0:
            result.put(out.numpy().tolist())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gather_operator_outputs_world_gloo(world):
    from oracle.oracle import OracleBatch
    from paper_1708_08427_b200.workloads import ellipsoid_batch

    pos, off = ellipsoid_batch([300, 1200, 64] if world == 2 else [500, 700], seed=9)  # world 3: one empty shard
    v = np.random.default_rng(3).normal(size=3 * int(off[-1]))
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_oracle_worker, args=(r, world, port, pos, off, v, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
        assert p.exitcode == 0
    got = np.array(q.get())
    want = OracleBatch(pos, off, threads=1).apply("qtilde_v", v)
    np.testing.assert_array_equal(got, want)  # per-body arithmetic does not depend on the split


def test_empty_shard_operator():
    """world > m: the empty rank builds nothing and returns zero-row outputs (no GPU needed)."""
    from paper_1708_08427_b200.parallel import ShardedMultiBodyOperator

    pos = np.random.default_rng(0).normal(size=(10, 3))
    off = np.array([0, 10])
    b = shard_bounds(off, 2)
    empty = 0 if b[1] == b[0] else 1
    sh = ShardedMultiBodyOperator(pos, off, rank=empty, world=2)
    assert sh.local is None and sh.j0 == sh.j1
    assert sh.apply("qtilde_v", np.zeros(0)).shape == (0,)
    assert sh.apply_global("qtilde_tv", np.zeros(30 - 6)).shape == (0,)
    with pytest.raises(ValueError):
        sh.apply("bad", np.zeros(0))
