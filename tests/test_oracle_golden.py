"""Pin the C oracle against the reference package's own outputs (tests/golden)."""

import numpy as np
import pytest

from conftest import GOLDEN, golden_cases

TREE_KEYS = ("perm", "start", "stop", "left", "right", "split_axis", "depth", "box",
             "case", "fn", "fnx", "fny", "swapped", "res_offsets")


def load(name):
    return dict(np.load(f"{GOLDEN}/{name}.npz"))


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


@pytest.mark.parametrize("name", golden_cases())
def test_oracle_tree_and_factors(oracle_mod, name):
    g = load(name)
    off = g["offsets"]
    degenerate = name.startswith("line")
    for j in range(len(off) - 1):
        ob = oracle_mod.OracleBody(g["positions"][off[j]:off[j + 1]])
        for key in TREE_KEYS:
            ours = getattr(ob, {"case": "case"}.get(key, key))
            np.testing.assert_array_equal(np.asarray(ours), g[f"b{j}_{key}"], err_msg=key)
        np.testing.assert_array_equal(ob.centroid, g[f"b{j}_centroid"])  # exact recursion
        assert ob.total_rows == int(g[f"b{j}_total_rows"])
        np.testing.assert_allclose(ob.t22, g[f"b{j}_t22"], rtol=0, atol=1e-12)
        if not degenerate:
            om = np.concatenate([o.ravel() for o in ob.omega if o is not None]) if ob.n > 1 else np.zeros(0)
            np.testing.assert_allclose(om, g[f"b{j}_omega"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("name", [c for c in golden_cases() if not c.startswith("line")])
def test_oracle_apply(oracle_mod, name):
    g = load(name)
    ob = oracle_mod.OracleBatch(g["positions"], g["offsets"], threads=2)
    for op, src in (("qv", "v"), ("qtv", "w"), ("qtilde_v", "v"), ("qtilde_tv", "g")):
        if op not in g:
            continue
        assert rel(ob.apply(op, g[src]), g[op]) < 1e-12, op
        ks = {"v": "V", "w": "W", "g": "G"}[src]
        assert rel(ob.apply(op, g[ks]), g[op + "_k"]) < 1e-12, op + "_k"
    if "zf" in g:
        zf = ob.zf(g["f"])
        # normalised by ||Z||_F ||f||_2
        m = len(g["offsets"]) - 1
        for j in range(m):
            o0, o1 = g["offsets"][j], g["offsets"][j + 1]
            p = g["positions"][o0:o1]
            zfro = np.sqrt(3 * (o1 - o0) + 2 * np.sum((p - p.mean(0)) ** 2))
            err = np.abs(zf[6 * j:6 * j + 6] - g["zf"][6 * j:6 * j + 6]).max()
            assert err <= 1e-13 * zfro * np.linalg.norm(g["f"][3 * o0:3 * o1])
        assert rel(ob.ztu(g["u"]), g["ztu"]) < 1e-13


def test_oracle_kat_pm(oracle_mod):
    """SPEC.md:265/345/355: beads +-(0,0,1), f=(1,0,0) twice -> Qv=(sqrt2,0,...)."""
    ob = oracle_mod.OracleBody(np.array([[0, 0, 1.0], [0, 0, -1.0]]))
    out = ob.qv(np.array([1.0, 0, 0, 1.0, 0, 0]))
    np.testing.assert_allclose(out, [np.sqrt(2), 0, 0, 0, 0, 0], atol=1e-15)
    back = ob.qtv(out)
    np.testing.assert_allclose(back, [1, 0, 0, 1, 0, 0], atol=1e-15)


def test_oracle_small_lq_kats(oracle_mod):
    """[I|0] -> (I, I); zero -> (0, I); random reconstructs."""
    a = np.hstack([np.eye(3), np.zeros((3, 6))])
    t, om = oracle_mod.small_lq(a)
    np.testing.assert_allclose(t, np.eye(3), atol=1e-15)
    np.testing.assert_allclose(om, np.eye(9), atol=1e-15)
    t, om = oracle_mod.small_lq(np.zeros((3, 9)))
    assert not t.any() and np.array_equal(om, np.eye(9))
    rng = np.random.default_rng(0)
    for k in (3, 6, 9):
        a = rng.normal(size=(3, k))
        t, om = oracle_mod.small_lq(a)
        rec = np.hstack([t, np.zeros((3, k - 3))]) @ om
        assert np.abs(rec - a).max() < 1e-13
        assert np.abs(om @ om.T - np.eye(k)).max() < 1e-14
        assert np.all(np.diag(t) >= 0) and np.allclose(np.triu(t, 1), 0)
