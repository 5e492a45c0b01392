"""Adaptive binary spatial tree of one body (tree.py:1-172 of the reference).

``build_tree`` runs the whole batched GPU setup (rq_setup: bounding cube,
ghost keys, radix sort, radix-tree topology, bottom-up factor pass, apply
layout) for one body; the returned BodyTree is a handle to the device-resident
tree.  ``nodes`` (TreeNode objects in postorder) and ``perm`` are exported
lazily for inspection and parity checks.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ._plan import Plan
from .model import BeadModel

_AXIS_CYCLE = (2, 1, 0)  # tree.py:27
DEFAULT_MAX_DEPTH = 96   # tree.py:29


@dataclass
class TreeNode:
    id: int
    start: int              # half-open bead range [start, stop) in tree order
    stop: int
    children: tuple | None  # (left_id, right_id) or None for a leaf
    centroid: np.ndarray
    box: np.ndarray         # (2, 3) lower/upper bounds of the node's cell
    split_axis: int | None  # axis of the final successful bisection
    depth: int              # ghost depth at which the node was created

    @property
    def n_beads(self) -> int:
        return self.stop - self.start

    @property
    def is_leaf(self) -> bool:
        return self.children is None


class BodyTree:
    """Handle to a device-resident tree (arena in postorder + bead permutation)."""

    def __init__(self, plan: Plan, body: int, positions_orig: np.ndarray):
        self._plan = plan
        self._body = body
        self._pos_orig = positions_orig
        self.n = int(plan.n[body])
        self.root_id = 2 * self.n - 2
        self._arrays = None
        self._nodes = None

    def _export(self):
        if self._arrays is None:
            self._arrays = self._plan.export_tree(self._body)
        return self._arrays

    @property
    def perm(self) -> np.ndarray:
        return self._export()["perm"]

    @property
    def positions(self) -> np.ndarray:
        return self._pos_orig[self.perm]

    @property
    def nodes(self) -> list:
        if self._nodes is None:
            a = self._export()
            nodes = []
            for i in range(2 * self.n - 1):
                leaf = a["left"][i] < 0
                nodes.append(TreeNode(
                    i, int(a["start"][i]), int(a["stop"][i]),
                    None if leaf else (int(a["left"][i]), int(a["right"][i])),
                    a["centroid"][i].copy(), a["box"][i].copy(),
                    None if leaf else int(a["split_axis"][i]), int(a["depth"][i])))
            self._nodes = nodes
        return self._nodes

    @property
    def root(self) -> TreeNode:
        return self.nodes[self.root_id]

    def depth(self) -> int:
        return int(self._export()["depth"].max())

    def __len__(self):
        return 2 * self.n - 1


def build_tree(model: BeadModel, max_depth: int = DEFAULT_MAX_DEPTH) -> BodyTree:
    """Build the binary spatial tree (and its factors) on the GPU (tree.py:73-134)."""
    plan = Plan(model.positions, np.array([0, model.n], np.int64), max_depth=max_depth)
    return BodyTree(plan, 0, model.positions)


def validate_tree(tree: BodyTree) -> list[str]:
    """Check the structural invariants; return a list of violations (tree.py:137-164)."""
    problems = []
    n = tree.n
    if len(tree.nodes) != 2 * n - 1:
        problems.append(f"node count {len(tree.nodes)} != 2n-1 = {2 * n - 1}")
    seen = np.sort(tree.perm)
    if tree.perm.shape != (n,) or not np.array_equal(seen, np.arange(n)):
        problems.append("perm is not a bijection on 0..n-1")
    positions = tree.positions
    for node in tree.nodes:
        if node.is_leaf:
            if node.n_beads != 1:
                problems.append(f"node {node.id}: leaf holds {node.n_beads} beads")
            continue
        left, right = node.children
        ln, rn = tree.nodes[left], tree.nodes[right]
        if node.n_beads != ln.n_beads + rn.n_beads:
            problems.append(f"node {node.id}: n_beads != sum of children")
        if (ln.start, rn.stop) != (node.start, node.stop) or ln.stop != rn.start:
            problems.append(f"node {node.id}: children do not tile its bead range")
        direct = positions[node.start:node.stop].mean(axis=0)
        scale = max(1.0, float(np.abs(positions).max()))
        if np.abs(node.centroid - direct).max() > 1e-13 * scale:
            problems.append(f"node {node.id}: centroid drifts from direct mean")
    return problems


def dump_tree(tree: BodyTree, fp) -> None:
    """One line per node: id n_beads centroid children (-1 for absent) (tree.py:167-172)."""
    for node in tree.nodes:
        c0, c1 = node.children if node.children else (-1, -1)
        cx, cy, cz = node.centroid
        fp.write(f"{node.id} {node.n_beads} {cx:.17g} {cy:.17g} {cz:.17g} {c0} {c1}\n")
