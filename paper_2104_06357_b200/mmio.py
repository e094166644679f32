"""Matrix Market ingest and result writers (reference:
/root/reference/pkg/src/semidist/mmio.py), the host I/O around the path.

``read_matrix_market`` parses a coordinate file (real / integer / pattern
field, general / symmetric storage) with the reference's error contract —
``ParseError`` carrying the 1-based line number, ``UnsupportedField`` for
formats it does not read — then hands the raw triple to the device
canonicalizer (``validate_and_canonicalize`` -> sd_canonicalize: sort,
duplicates summed in file order, zeros dropped).  Entry lines are converted
in bulk with numpy; only a line that fails the bulk conversion is re-scanned
to name it.  Floats are written with 17 significant digits, so a
write/read round trip is bitwise exact.
"""

import json

import numpy as np

from .errors import ParseError, UnsupportedField
from .knn import NeighborResult
from .sparse import validate_and_canonicalize

_FIELDS = ("real", "integer", "pattern")
_SYMMETRY = ("general", "symmetric")


def _g17(v):
    return f"{v:.17g}"


def _content(lines, start):
    """(line number, text) of the non-blank, non-comment lines from index `start`."""
    for i in range(start, len(lines)):
        text = lines[i].strip()
        if text and not text.startswith("%"):
            yield i + 1, text


def _header(first):
    parts = first.strip().split()
    if len(parts) < 5 or parts[0].lower() != "%%matrixmarket":
        raise ParseError(1, "missing MatrixMarket header")
    obj, layout, field, symmetry = (t.lower() for t in parts[1:5])
    if obj != "matrix":
        raise UnsupportedField(f"object '{obj}' not supported")
    if layout != "coordinate":
        raise UnsupportedField(f"format '{layout}' not supported (coordinate only)")
    if field not in _FIELDS:
        raise UnsupportedField(f"field '{field}' not supported")
    if symmetry not in _SYMMETRY:
        raise UnsupportedField(f"symmetry '{symmetry}' not supported")
    return field, symmetry


def _entries(numbered, declared, want, pattern, n_rows, n_cols, last_line):
    """Bulk-convert the entry lines; on any failure, locate the first bad line."""
    extra = numbered[declared] if len(numbered) > declared else None
    numbered = numbered[:declared]
    toks = [t.split() for _, t in numbered]
    try:
        if any(len(t) != want for t in toks):
            raise ValueError
        arr = np.array(toks, dtype=object).reshape(len(toks), want) if toks else np.empty((0, want), dtype=object)
        rows = arr[:, 0].astype(np.int64) if toks else np.empty(0, dtype=np.int64)
        cols = arr[:, 1].astype(np.int64) if toks else np.empty(0, dtype=np.int64)
        vals = np.ones(len(toks)) if pattern else (arr[:, 2].astype(np.float64) if toks else np.empty(0))
        bad = (rows < 1) | (rows > n_rows) | (cols < 1) | (cols > n_cols)
        if bad.any():
            raise ValueError
    except (ValueError, TypeError, OverflowError):
        for (line_no, text), t in zip(numbered, toks):   # name the first offending line
            if len(t) != want:
                raise ParseError(line_no, f"expected {want} fields, found {len(t)}") from None
            try:
                i, j = int(t[0]), int(t[1])
                if not pattern:
                    float(t[2])
            except ValueError:
                raise ParseError(line_no, f"malformed entry '{text}'") from None
            if not (1 <= i <= n_rows and 1 <= j <= n_cols):
                raise ParseError(line_no, f"entry ({i}, {j}) outside {n_rows} x {n_cols}") from None
        raise
    if extra is not None:
        raise ParseError(extra[0], f"more than the declared {declared} entries")
    if len(numbered) < declared:
        raise ParseError(last_line, f"declared {declared} entries, found {len(numbered)}")
    return rows - 1, cols - 1, vals


def read_matrix_market(path, *, device=None):
    """Parse a Matrix Market coordinate file into a canonical CSR matrix."""
    with open(path, "r", encoding="utf-8") as fh:
        lines = fh.read().split("\n")
    if len(lines) == 1 and lines[0] == "":
        raise ParseError(1, "empty file")
    field, symmetry = _header(lines[0])
    body = _content(lines, 1)
    size = next(body, None)
    if size is None:
        raise ParseError(len(lines) - (1 if lines[-1] == "" else 0), "missing size line")
    size_no, size_text = size
    tokens = size_text.split()
    if len(tokens) != 3:
        raise ParseError(size_no, "size line must be 'rows cols nnz'")
    try:
        n_rows, n_cols, declared = (int(t) for t in tokens)
    except ValueError:
        raise ParseError(size_no, "size line must contain integers") from None
    if min(n_rows, n_cols, declared) < 0:
        raise ParseError(size_no, "sizes must be non-negative")
    if symmetry == "symmetric" and n_rows != n_cols:
        raise ParseError(size_no, "symmetric storage requires a square matrix")
    numbered = list(body)
    last_line = len(lines) - (1 if lines[-1] == "" else 0)
    pattern = field == "pattern"
    rows, cols, vals = _entries(numbered, declared, 2 if pattern else 3, pattern, n_rows, n_cols, last_line)
    if symmetry == "symmetric" and rows.size:
        off = rows != cols
        rows, cols = np.concatenate([rows, cols[off]]), np.concatenate([cols, rows[off]])
        vals = np.concatenate([vals, vals[off]])
    # group by row (stable: duplicates keep file order); columns are sorted and
    # duplicates summed on the device
    order = np.argsort(rows, kind="stable")
    indptr = np.zeros(n_rows + 1, dtype=np.int64)
    if rows.size:
        np.cumsum(np.bincount(rows, minlength=n_rows), out=indptr[1:])
    return validate_and_canonicalize(indptr, cols[order], vals[order], n_cols=n_cols, n_rows=n_rows, device=device)


def write_matrix_market(m, path):
    """CSR matrix -> 'coordinate real general', 1-based ids, 17 significant digits."""
    deg = np.diff(np.asarray(m.indptr))
    rows = np.repeat(np.arange(1, m.n_rows + 1), deg)
    body = "".join(f"{r} {c} {_g17(v)}\n" for r, c, v in
                   zip(rows.tolist(), (np.asarray(m.indices) + 1).tolist(), np.asarray(m.values).tolist()))
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("%%MatrixMarket matrix coordinate real general\n")
        fh.write(f"{m.n_rows} {m.n_cols} {m.nnz}\n")
        fh.write(body)


def write_output(result, path, fmt="csv", header=False):
    """A distance matrix or a NeighborResult as CSV or JSON (mmio.py:112-162 formats)."""
    if fmt not in ("csv", "json"):
        raise ValueError(f"unsupported output format '{fmt}'")
    knn = isinstance(result, NeighborResult) or (hasattr(result, "indices") and hasattr(result, "distances"))
    with open(path, "w", encoding="utf-8") as fh:
        if knn:
            ids, dist = np.asarray(result.indices), np.asarray(result.distances, dtype=np.float64)
            if fmt == "json":
                json.dump([{"query_id": q, "neighbor_id": int(j), "distance": float(d)}
                           for q in range(ids.shape[0]) for j, d in zip(ids[q].tolist(), dist[q].tolist())], fh)
                fh.write("\n")
                return
            if header:
                fh.write("query_id,neighbor_id,distance\n")
            fh.write("".join(f"{q},{j},{_g17(d)}\n" for q in range(ids.shape[0])
                             for j, d in zip(ids[q].tolist(), dist[q].tolist())))
            return
        mat = np.asarray(result, dtype=np.float64)
        if fmt == "json":
            json.dump({"n_rows": mat.shape[0], "n_cols": mat.shape[1], "distances": mat.tolist()}, fh)
            fh.write("\n")
            return
        if header:
            fh.write(",".join(f"j{c}" for c in range(mat.shape[1])) + "\n")
        fh.write("".join(",".join(_g17(v) for v in row) + "\n" for row in mat.tolist()))
