"""Multi-GPU sharding of independent rigid bodies.

Bodies are independent (Q~ and Z are block diagonal, matfree.py:212-216), so
a batch is split contiguously in body order into ``world`` shards of nearly
equal bead count.  Every rank builds and applies the operator of its own shard
only -- there is no collective on the data path.  ``gather_shards`` is the one
collective: it concatenates per-rank outputs in body order on every rank (or
on rank 0), with torch.distributed (NCCL over NVLink on GPUs; gloo in the CPU
tests).  Because the layout is contiguous, the global output is a plain
concatenation of the shard outputs.
"""

from __future__ import annotations

import numpy as np


def shard_bounds(offsets, world: int) -> np.ndarray:
    """Body-index cut points (world+1,) splitting bodies by cumulative bead count.

    Shard r owns bodies [b[r], b[r+1]).  Cuts are chosen at the body boundary
    nearest to r * N / world, so the imbalance is bounded by one body.
    """
    offsets = np.asarray(offsets, dtype=np.int64)
    m = len(offsets) - 1
    if world < 1:
        raise ValueError("world must be >= 1")
    N = int(offsets[-1])
    cuts = [0]
    for r in range(1, world):
        target = r * N / world
        j = int(np.searchsorted(offsets, target))
        if j > 0 and (j > m or abs(offsets[j - 1] - target) <= abs(offsets[j] - target)):
            j -= 1
        j = min(max(j, cuts[-1]), m)
        cuts.append(j)
    cuts.append(m)
    return np.asarray(cuts, dtype=np.int64)


def shard_of(positions, offsets, rank: int, world: int):
    """(positions, offsets) of this rank's shard (offsets rebased to 0)."""
    offsets = np.asarray(offsets, dtype=np.int64)
    b = shard_bounds(offsets, world)
    j0, j1 = int(b[rank]), int(b[rank + 1])
    lo, hi = int(offsets[j0]), int(offsets[j1])
    return np.asarray(positions)[lo:hi], offsets[j0:j1 + 1] - lo, (j0, j1)


def vector_slice(offsets, bounds, rank: int, kind: str):
    """Row range of shard ``rank`` inside a global vector.

    kind: "full" (3N rows: Qv / Q^T w / Q~^T g outputs, Zf inputs...),
          "comp" (3N - 6m rows: Q~ coefficients), "body6" (6m rows: Zf outputs).
    """
    offsets = np.asarray(offsets, dtype=np.int64)
    j0, j1 = int(bounds[rank]), int(bounds[rank + 1])
    if kind == "full":
        return 3 * int(offsets[j0]), 3 * int(offsets[j1])
    if kind == "comp":
        return 3 * int(offsets[j0]) - 6 * j0, 3 * int(offsets[j1]) - 6 * j1
    if kind == "body6":
        return 6 * j0, 6 * j1
    raise ValueError(f"unknown vector kind {kind!r}")


def gather_shards(local, rows_per_rank, group=None):
    """Concatenate every rank's ``local`` (rows, ...) tensor in rank order.

    Uses all_gather over max-padded buffers (one collective); works with the
    NCCL (CUDA tensors) and gloo (CPU tensors) backends.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rows = [int(r) for r in rows_per_rank]
    if len(rows) != world:
        raise ValueError("rows_per_rank must have one entry per rank")
    pad = max(rows) if rows else 0
    shape = (pad,) + tuple(local.shape[1:])
    buf = torch.zeros(shape, dtype=local.dtype, device=local.device)
    buf[: local.shape[0]] = local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return torch.cat([p[:r] for p, r in zip(parts, rows)], dim=0)


class ShardedMultiBodyOperator:
    """This rank's share of a MultiBodyOperator (one process per GPU).

    ``apply(op, v_local)`` applies the operator to the rank's own slice;
    ``gather(op, out_local)`` reassembles the global result (the only
    collective).  Inputs of ``apply_global`` are full global vectors.
    """

    def __init__(self, positions, offsets, rank: int, world: int, max_depth: int = 96):
        from .matfree import MultiBodyOperator
        from .model import MultiBodyModel

        self.offsets = np.asarray(offsets, dtype=np.int64)
        self.rank, self.world = rank, world
        self.bounds = shard_bounds(self.offsets, world)
        pos, off, (self.j0, self.j1) = shard_of(positions, self.offsets, rank, world)
        # more ranks than bodies (or one body dominating) leaves a shard empty: it applies
        # nothing and contributes zero rows to the gather
        self.local = (MultiBodyOperator(MultiBodyModel.from_arrays(pos, off), max_depth=max_depth)
                      if self.j1 > self.j0 else None)

    def _kinds(self, op):
        return {"qv": ("full", "full"), "qtv": ("full", "full"), "qtilde_v": ("full", "comp"),
                "qtilde_tv": ("comp", "full")}[op]

    def local_rows(self, kind: str, rank: int | None = None):
        a, b = vector_slice(self.offsets, self.bounds, self.rank if rank is None else rank, kind)
        return a, b

    def apply(self, op: str, v_local):
        if self.local is None:
            if op not in ("qv", "qtv", "qtilde_v", "qtilde_tv"):
                raise ValueError("op must be one of ('qv', 'qtv', 'qtilde_v', 'qtilde_tv')")
            return v_local[:0]
        return self.local.apply(op, v_local)

    def apply_global(self, op: str, v):
        kin, _ = self._kinds(op)
        a, b = self.local_rows(kin)
        return self.apply(op, v[a:b])

    def gather(self, op: str, out_local, group=None):
        _, kout = self._kinds(op)
        rows = [vector_slice(self.offsets, self.bounds, r, kout) for r in range(self.world)]
        return gather_shards(out_local, [b - a for a, b in rows], group=group)
