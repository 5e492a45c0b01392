"""GPU dense validation tools (validation.py, the reference's oracle.py:38-270): the dense
complement of Z (cuSOLVER SVD) spans the same space as the hierarchical Q~ (projector
distance ~1e-15), and the per-body orthogonality report matches the reference's columns."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_dense_complement_and_report():
    import paper_1708_08427_b200 as rq
    from paper_1708_08427_b200 import validation as V
    from paper_1708_08427_b200.workloads import make_config

    pos, _ = make_config(1, seed=0)
    model = rq.BeadModel(pos)
    n = model.n
    dc = V.dense_complement(rq.assemble_z(model))
    assert dc.rank == 6 and dc.qtilde.shape == (3 * n - 6, 3 * n)
    qt = rq.BodyOperator(model).qtilde_v(np.eye(3 * n))
    assert V.projector_distance(qt, dc.qtilde) < 1e-12
    assert V.max_abs_gram_deviation(qt) < 1e-12
    row = V.body_report(rq.BeadModel(pos[:700]), seed=3)
    assert row["n"] == 700 and all(row[c] < 1e-12 for c in V.REPORT_COLUMNS[1:])
    csv = V.report_to_csv([row, V.body_report(rq.BeadModel(pos[:1]))])
    lines = csv.splitlines()
    assert lines[0] == ",".join(V.REPORT_COLUMNS) and lines[2] == "1," + ",".join(["na"] * 6)
    with pytest.raises(rq.SizeGuardError):
        V.dense_complement(np.zeros((6, 9000)))
