"""Text wire formats on either side of the hot path (reference io.py:1-72).

* Bead file: one bead per line, three whitespace-separated decimals (written
  with 17 significant digits, so values round-trip exactly); lines starting
  with '#' and blank lines are skipped; a line holding only '---' separates
  bodies (io.py:18-44).
* Vector file: one decimal per line; a spectral vector (Qv layout) carries the
  header '# spectral n=<n>' (io.py:47-72).

Output is byte-identical to the reference's writers and the readers raise the
same ValueError messages (tests/test_io.py pins both against files the
reference itself wrote, tests/golden/io_*).  These are host-side text
conversions; the bodies a bead file describes are validated (finite,
duplicate-free) by the batched GPU check of ``MultiBodyModel``.
"""

from __future__ import annotations

import numpy as np

from .model import BeadModel, MultiBodyModel

_FMT = "{:.17g}"


def _lines_of_rows(rows: np.ndarray) -> str:
    fmt = " ".join([_FMT] * rows.shape[1]) + "\n"
    return "".join(fmt.format(*r) for r in rows.tolist())


def save_beads(model, fp) -> None:
    """Write one body or a multi-body model; bodies are separated by '---' (io.py:18-24)."""
    if isinstance(model, MultiBodyModel):
        pos, off = np.asarray(model.positions, dtype=float), model.offsets
    else:
        pos = np.asarray(model.positions, dtype=float)
        off = np.array([0, pos.shape[0]], np.int64)
    parts = [_lines_of_rows(pos[off[j]:off[j + 1]]) for j in range(len(off) - 1)]
    fp.write("---\n".join(parts))


def parse_beads(fp):
    """Parse a bead file into (positions (n, 3), offsets (m + 1,), body_ids (m,)).

    Empty bodies (e.g. a leading '---') are dropped but still advance the body id,
    as the reference's ``enumerate(chunks) if c`` does (io.py:27-44)."""
    coords: list[list[float]] = []
    counts = [0]
    for lineno, line in enumerate(fp, 1):
        s = line.strip()
        if not s or s[0] == "#":
            continue
        if s == "---":
            counts.append(0)
            continue
        fields = s.split()
        if len(fields) != 3:
            raise ValueError(f"line {lineno}: expected 3 coordinates, got {len(fields)}")
        try:
            coords.append([float(f) for f in fields])
        except ValueError as exc:
            raise ValueError(f"line {lineno}: {exc}") from None
        counts[-1] += 1
    counts = np.asarray(counts, dtype=np.int64)
    keep = np.nonzero(counts)[0]
    if keep.size == 0:
        raise ValueError("no beads found")
    offsets = np.concatenate([[0], np.cumsum(counts[keep])]).astype(np.int64)
    return np.asarray(coords, dtype=float).reshape(-1, 3), offsets, keep.astype(np.int64)


def load_beads(fp) -> MultiBodyModel:
    """Read a bead file into a MultiBodyModel (io.py:27-44); every body goes through the
    BeadModel validation (finite positions, duplicate beads) in one batched GPU check."""
    pos, offsets, ids = parse_beads(fp)
    checked = MultiBodyModel.from_arrays(pos, offsets)  # finite + duplicate check, all bodies at once
    return MultiBodyModel([BeadModel(checked.positions[offsets[j]:offsets[j + 1]], body_id=int(ids[j]),
                                     check_duplicates=False) for j in range(len(ids))])


def save_vector(vec, fp, spectral_n: int | None = None) -> None:
    """One value per line, '# spectral n=<n>' header for spectral vectors (io.py:47-51)."""
    if hasattr(vec, "detach"):  # torch tensors (CUDA or host)
        vec = vec.detach().cpu().numpy()
    if spectral_n is not None:
        fp.write(f"# spectral n={spectral_n}\n")
    flat = np.asarray(vec, dtype=float).ravel()
    fp.write("".join(f"{x:.17g}\n" for x in flat.tolist()))


def load_vector(fp) -> tuple[np.ndarray, int | None]:
    """Returns (vector, spectral_n or None) (io.py:54-72)."""
    vals: list[float] = []
    spectral_n = None
    for lineno, line in enumerate(fp, 1):
        s = line.strip()
        if not s:
            continue
        if s[0] == "#":
            if s.startswith("# spectral n="):
                spectral_n = int(s.split("=", 1)[1])
            continue
        try:
            vals.append(float(s))
        except ValueError:
            raise ValueError(f"line {lineno}: not a number: {s!r}") from None
    return np.array(vals), spectral_n
