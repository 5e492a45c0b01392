"""Generate the text-format fixtures (tests/golden/io/) with the reference's own io.py.

Runs ONLY in the build container, where the reference is importable:

    python tests/golden/make_io_golden.py

Writes the files the reference's writers produce (bead file, plain and spectral
vector files), the positions / vectors its readers return for a hand-written
input with comments, blank lines and empty bodies, and the ValueError messages
its readers raise for malformed lines.
"""

from __future__ import annotations

import io
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "io")
sys.path.insert(0, "/root/reference/pkg/src")

import rigidq as R  # noqa: E402  (the reference package)
from rigidq import io as RIO  # noqa: E402


def main():
    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(11)
    bodies = [rng.normal(size=(5, 3)), rng.normal(size=(1, 3)) * 1e-300, rng.normal(size=(7, 3)) * 1e12]
    bodies[0][0] = [-0.0, 1.0, 2.5]
    bodies[2][3] = [1 / 3, -2 / 3, 1e-5]
    model = R.MultiBodyModel([R.BeadModel(b, body_id=j) for j, b in enumerate(bodies)])
    buf = io.StringIO()
    RIO.save_beads(model, buf)
    open(os.path.join(OUT, "beads_written.txt"), "w").write(buf.getvalue())
    buf = io.StringIO()
    RIO.save_beads(R.BeadModel(bodies[0]), buf)
    open(os.path.join(OUT, "beads_single_written.txt"), "w").write(buf.getvalue())

    op = R.BodyOperator(R.BeadModel(bodies[2]))
    v = rng.normal(size=3 * 7)
    qv = op.qv(v)
    buf = io.StringIO()
    RIO.save_vector(qv, buf, spectral_n=7)
    open(os.path.join(OUT, "vector_spectral_written.txt"), "w").write(buf.getvalue())
    buf = io.StringIO()
    RIO.save_vector(v, buf)
    open(os.path.join(OUT, "vector_plain_written.txt"), "w").write(buf.getvalue())
    np.save(os.path.join(OUT, "vector_values.npy"), np.stack([v, qv]))

    messy = ("# a comment\n---\n\n0 0 0\n 1 0 0 \n# body break follows\n---\n---\n"
             "0.5 0.25 -1e-3\n2 2 2\n1e2 -0 3\n---\n")
    open(os.path.join(OUT, "beads_messy.txt"), "w").write(messy)
    m = RIO.load_beads(io.StringIO(messy))
    parsed = {"positions": np.concatenate([b.positions for b in m.bodies]).tolist(),
              "counts": [b.n for b in m.bodies], "body_ids": [b.body_id for b in m.bodies]}
    vec_text = "# spectral n=4\n1.5\n\n-2\n# other comment\n3e-7\n"
    vals, sn = RIO.load_vector(io.StringIO(vec_text))
    parsed["vector_text"] = vec_text
    parsed["vector"] = vals.tolist()
    parsed["spectral_n"] = sn
    errors = {}
    for name, text, fn in [("two_coords", "0 0 0\n1 2\n", RIO.load_beads),
                           ("bad_float", "0 0 0\n1 x 2\n", RIO.load_beads),
                           ("empty", "# nothing\n---\n", RIO.load_beads),
                           ("bad_value", "1\n2\nabc\n", RIO.load_vector)]:
        try:
            fn(io.StringIO(text))
            errors[name] = [text, None]
        except ValueError as exc:
            errors[name] = [text, str(exc)]
    parsed["errors"] = errors
    json.dump(parsed, open(os.path.join(OUT, "parsed.json"), "w"), indent=1)

    # text dumps of a tree (tree.py:167-172) and of the explicit Q (factor.py:351-359)
    from rigidq.factor import generate_explicit_q
    from rigidq.tree import build_tree, dump_tree

    pos = np.random.default_rng(12).normal(size=(40, 3))
    np.save(os.path.join(OUT, "dump_positions.npy"), pos)
    tree = build_tree(R.BeadModel(pos))
    buf = io.StringIO()
    dump_tree(tree, buf)
    open(os.path.join(OUT, "tree_dump.txt"), "w").write(buf.getvalue())
    buf = io.StringIO()
    generate_explicit_q(tree).dump(buf)
    open(os.path.join(OUT, "hierq_dump.txt"), "w").write(buf.getvalue())


if __name__ == "__main__":
    main()
