"""CPU-side checks: the C-ABI library loads and exports every symbol the
header declares; host-side validation and error mapping; the product path
fails loudly without a GPU (no CPU fallback)."""

import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "rigidq_b200.h")
LIB = os.path.join(ROOT, "paper_1708_08427_b200", "librigidq_b200.so")


@pytest.fixture(scope="module")
def built():
    if not os.path.exists(LIB):
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "paper_1708_08427_b200", "csrc")], check=True)
    return LIB


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const char \*|int64_t |int )(rq_\w+)\(", text, re.M)))


def test_header_symbols_exported(built):
    out = subprocess.run(["nm", "-D", "--defined-only", built], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (rq_\w+)", out))
    decl = declared_symbols()
    assert len(decl) >= 20
    missing = [s for s in decl if s not in exported]
    assert not missing, missing


def test_ctypes_binds_every_symbol(built):
    from paper_1708_08427_b200 import _lib

    L = _lib.lib()
    bound = {name for name, _, _ in _lib.SIGNATURES}
    assert bound == set(declared_symbols())
    for name in bound:
        assert getattr(L, name) is not None
    assert L.rq_version() >= 100


def test_no_gpu_fails_loudly(built):
    from paper_1708_08427_b200 import _lib

    import paper_1708_08427_b200 as rq

    if _lib.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        rq.BeadModel([[0, 0, 0], [1, 1, 1]])
    with pytest.raises(RuntimeError):
        rq.small_lq(np.eye(3))


def test_host_validation(built):
    import paper_1708_08427_b200 as rq

    with pytest.raises(ValueError, match="finite"):
        rq.BeadModel([[0, 0, np.inf]])
    with pytest.raises(ValueError, match=r"\(n, 3\)"):
        rq.BeadModel(np.zeros((4, 2)))
    with pytest.raises(ValueError):
        rq.MultiBodyModel([])
    with pytest.raises(ValueError):
        rq.MultiBodyModel.from_arrays(np.zeros((4, 3)), [0, 2, 2, 4], check_duplicates=False)
    # single-bead model skips the (GPU) duplicate check, like the reference (model.py:66-68)
    m = rq.BeadModel([[1.0, 2.0, 3.0]])
    assert m.n == 1 and np.array_equal(rq.centroid(m), [1, 2, 3])
    np.testing.assert_array_equal(rq.skew([1, 2, 3]), [[0, -3, 2], [3, 0, -1], [-2, 1, 0]])
    z = rq.assemble_z(rq.BeadModel([[0.0, 0.0, 1.0]]), origin=np.zeros(3)).entries
    np.testing.assert_array_equal(z[:3], np.eye(3))
    np.testing.assert_array_equal(z[3:], rq.skew([0, 0, 1]))


def test_public_names_match_reference(built):
    """Every hot-path name of the reference's __all__ (__init__.py:34-53) exists here."""
    import paper_1708_08427_b200 as rq

    names = ["BeadModel", "MultiBodyModel", "ZMatrix", "assemble_z", "centroid", "skew", "BodyTree", "TreeNode",
             "build_tree", "validate_tree", "dump_tree", "NodeCase", "NodeFactor", "FactorTable", "HierQ",
             "small_lq", "child_shift", "mean_block", "factor_leaf", "factor_bead_bead", "factor_rigid_bead",
             "factor_general", "factor_all", "node_rows", "generate_explicit_q", "materialize_dense",
             "leaf_infoset", "merge_infosets", "split_rvset", "upward_apply", "downward_apply", "qtilde_apply",
             "qtilde_transpose_apply", "multibody_apply", "BodyOperator", "MultiBodyOperator", "RigidQError",
             "DuplicateBeadsError", "TooSmallError", "SizeGuardError", "LengthMismatchError",
             "BodyTooSmallError", "ShapeMismatchError", "SingularHError", "load_beads", "save_beads",
             "load_vector", "save_vector", "RigidBodyBasis"]
    for n in names:
        assert hasattr(rq, n), n


def test_workload_generators():
    from paper_1708_08427_b200.workloads import config4_counts, ellipsoid_batch, sphere_shell

    p = sphere_shell(1024, 0)
    assert p.shape == (1024, 3) and np.abs(p.mean(0)).max() < 1e-15
    r = np.linalg.norm(p + 0, axis=1)
    assert 0.9 < r.mean() < 1.1
    pos, off = ellipsoid_batch([10, 20], seed=1)
    assert pos.shape == (30, 3) and list(off) == [0, 10, 30]
    c = config4_counts(m=20000)
    assert c.min() >= 500 and c.max() < 50000 and 1.9e8 < c.sum() < 2.4e8


def test_rigid_body_basis_validation():
    """Shape / finiteness checks of the estimator run before any GPU work."""
    from paper_1708_08427_b200.estimator import RigidBodyBasis

    with pytest.raises(ValueError, match="shape"):
        RigidBodyBasis().fit(np.zeros((4, 2)))
    with pytest.raises(ValueError, match="finite"):
        RigidBodyBasis().fit(np.array([[0.0, 0.0, np.nan], [1.0, 0.0, 0.0]]))


def test_c_abi_host_program_builds(built):
    """A plain C program compiles and links against include/rigidq_b200.h and
    librigidq_b200.so (tests/c_abi; run on the GPU by test_gpu_parity.test_c_abi_host_program)."""
    import subprocess

    r = subprocess.run(["make", "-s", "-B", "-C", os.path.join(ROOT, "tests", "c_abi")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert os.path.exists(os.path.join(ROOT, "tests", "c_abi", "c_abi_check"))
