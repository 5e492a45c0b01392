"""Seeded synthetic bead clouds for the BASELINE.json configurations.

These are the benchmark/test input generators; they are
not the reference's clouds.py kinds (which have no jitter and no centroid
shift).  Choices for the ambiguous parts of BASELINE.json are recorded in
DESIGN.md: "N(0,0.01)" is read as sigma = 0.01, and "uniform in surface
parameterisation" as (theta, phi) ~ U[0,pi] x U[0,2pi).
"""

from __future__ import annotations

import numpy as np


def sphere_shell(n: int, seed: int = 0) -> np.ndarray:
    """Config 1/3: unit-sphere directions x (1 + N(0, 0.01)), centroid-shifted."""
    rng = np.random.default_rng(seed)
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    p = d * (1.0 + 0.01 * rng.normal(size=(n, 1)))
    return p - p.mean(axis=0)


def _rotation(rng) -> np.ndarray:
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    return np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
        [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
        [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)],
    ])


def ellipsoid_shell(n: int, rng) -> np.ndarray:
    """Config 2/4/5 body: triaxial ellipsoid shell, semi-axes U[0.5, 2],
    beads uniform in (theta, phi), random rotation, centroid-shifted."""
    axes = rng.uniform(0.5, 2.0, size=3)
    th = rng.uniform(0.0, np.pi, size=n)
    ph = rng.uniform(0.0, 2.0 * np.pi, size=n)
    st = np.sin(th)
    p = np.stack([axes[0] * st * np.cos(ph), axes[1] * st * np.sin(ph), axes[2] * np.cos(th)], axis=1)
    p = p @ _rotation(rng).T
    return p - p.mean(axis=0)


def ellipsoid_batch(counts, seed: int = 0):
    """Concatenated positions (N, 3) and offsets (m+1,) for bodies of the given sizes."""
    counts = np.asarray(counts, dtype=np.int64)
    rng = np.random.default_rng(seed)
    offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    pos = np.empty((int(offsets[-1]), 3))
    for j, n in enumerate(counts):
        pos[offsets[j]:offsets[j + 1]] = ellipsoid_shell(int(n), rng)
    return pos, offsets


def config4_counts(m: int = 20000, seed: int = 0) -> np.ndarray:
    """Config 4: n_j = floor(exp(U[ln 500, ln 50000]))."""
    rng = np.random.default_rng([seed, 4])
    return np.floor(np.exp(rng.uniform(np.log(500.0), np.log(50000.0), size=m))).astype(np.int64)


CONFIGS = {
    1: dict(workload="cfg1: 1 sphere-shell body, n=1024", counts=[1024], kind="sphere"),
    2: dict(workload="cfg2: 1000 ellipsoid-shell bodies x 4096 beads", counts=[4096] * 1000, kind="ellipsoid"),
    3: dict(workload="cfg3: 1 sphere-shell body, n=2^20", counts=[1 << 20], kind="sphere"),
    5: dict(workload="cfg5: 2000 ellipsoid bodies x 8192 beads, k=32 RHS", counts=[8192] * 2000,
            kind="ellipsoid", k=32),
}


def make_config(cfg: int, seed: int = 0, scale: float = 1.0):
    """(positions, offsets) for a BASELINE config; ``scale`` < 1 shrinks the body count."""
    if cfg == 4:
        counts = config4_counts(seed=seed)
        counts = counts[: max(1, int(len(counts) * scale))]
        return ellipsoid_batch(counts, seed)
    spec = CONFIGS[cfg]
    counts = spec["counts"]
    if len(counts) > 1:
        counts = counts[: max(1, int(len(counts) * scale))]
    if spec["kind"] == "sphere":
        pos = sphere_shell(counts[0], seed)
        return pos, np.array([0, counts[0]], dtype=np.int64)
    return ellipsoid_batch(counts, seed)
