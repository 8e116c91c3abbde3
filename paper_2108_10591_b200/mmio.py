"""Matrix Market ingest for the device solvers (drop-in for pipesafe.mmio).

Same entry points, accepted formats and error behaviour as the reference
(mmio.py:33-151): coordinate ``real``/``integer`` matrices, ``general`` or
``symmetric`` (one stored triangle, mirrored on load), 1-based indices on
disk, duplicates summed through ``csr_from_coo`` (linalg.py:110-139), and a
``MatrixMarketError`` that names ``path:line`` of the offending line.  The
result is the canonical host CSR that ``DeviceMatrix.from_csr`` uploads
(int64 indices narrowed to int32 on the device).

The parse is one tokenisation of the entry block: every entry line must hold
exactly three tokens, so the block converts with a single numpy call and the
per-line checks only run to name the line of a failure.
"""

from __future__ import annotations

import numpy as np

from .linalg import CsrMatrix, MatrixMetadata, csr_from_coo

FIELDS = ("real", "integer")
SYMMETRIES = ("general", "symmetric")


class MatrixMarketError(ValueError):
    """Malformed or unsupported Matrix Market content (mmio.py:19-27)."""

    def __init__(self, message: str, path: str = "", line: int | None = None):
        if line is not None:
            prefix = f"{path}:{line}: "
        elif path:
            prefix = f"{path}: "
        else:
            prefix = ""
        super().__init__(prefix + message)
        self.path = path
        self.line = line


def _content_lines(lines, start):
    """(1-based line number, stripped text) of non-blank, non-comment lines."""
    for k in range(start, len(lines)):
        text = lines[k].strip()
        if text and not text.startswith("%"):
            yield k + 1, text


def _parse_banner(first: str, path: str) -> tuple[str, bool]:
    words = first.strip().lower().split()
    if len(words) != 5 or words[0] != "%%matrixmarket":
        raise MatrixMarketError("missing %%MatrixMarket header", path, 1)
    obj, fmt, field, symmetry = words[1:]
    if obj != "matrix":
        raise MatrixMarketError(f"unsupported object {obj!r}", path, 1)
    if fmt != "coordinate":
        raise MatrixMarketError(f"unsupported format {fmt!r} (need coordinate)", path, 1)
    if field not in FIELDS:
        raise MatrixMarketError(f"unsupported field {field!r} (need real/integer)", path, 1)
    if symmetry not in SYMMETRIES:
        raise MatrixMarketError(f"unsupported symmetry {symmetry!r} (need general/symmetric)", path, 1)
    return field, symmetry == "symmetric"


def _parse_sizes(lineno: int, text: str, path: str) -> tuple[int, int, int]:
    tokens = text.split()
    if len(tokens) != 3:
        raise MatrixMarketError("size line must be 'rows cols nnz'", path, lineno)
    try:
        sizes = tuple(int(t) for t in tokens)
    except ValueError:
        raise MatrixMarketError("non-integer size line", path, lineno) from None
    if min(sizes) < 0:
        raise MatrixMarketError("negative dimension on size line", path, lineno)
    return sizes


def _entry_table(entries, path: str) -> np.ndarray:
    """(n, 3) float64 table of the entry lines, or the error naming the bad line."""
    counts = [len(text.split()) for _, text in entries]
    for (lineno, _), c in zip(entries, counts):
        if c != 3:
            raise MatrixMarketError("entry must be 'row col value'", path, lineno)
    try:
        return np.array(" ".join(text for _, text in entries).split(), dtype=np.float64).reshape(-1, 3)
    except ValueError:
        pass
    for lineno, text in entries:
        a, b, v = text.split()
        try:
            int(float(a)), int(float(b)), float(v)
        except ValueError:
            raise MatrixMarketError(f"unparseable entry {text!r}", path, lineno) from None
    raise MatrixMarketError("unparseable entry", path, entries[0][0] if entries else 1)


def load_matrix_market(path: str) -> tuple[CsrMatrix, MatrixMetadata]:
    """Read a coordinate Matrix Market file into canonical CSR (mmio.py:33-137)."""
    with open(path, "r", encoding="ascii", errors="replace") as fh:
        lines = fh.read().splitlines()
    if not lines:
        raise MatrixMarketError("empty file", path, 1)
    _, symmetric = _parse_banner(lines[0], path)
    body = _content_lines(lines, 1)
    size = next(body, None)
    if size is None:
        raise MatrixMarketError("missing size line", path, len(lines))
    size_lineno = size[0]
    n_rows, n_cols, n_entries = _parse_sizes(*size, path)
    entries = list(body)
    if len(entries) != n_entries:
        raise MatrixMarketError(f"size line promises {n_entries} entries, file holds {len(entries)}",
                                path, size_lineno)
    if entries:
        table = _entry_table(entries, path)
        ri, ci, vals = table[:, 0], table[:, 1], table[:, 2]
        frac = (ri != np.floor(ri)) | (ci != np.floor(ci))
        if frac.any():
            raise MatrixMarketError("non-integer index", path, entries[int(np.argmax(frac))][0])
        rows = ri.astype(np.int64) - 1
        cols = ci.astype(np.int64) - 1
        outside = (rows < 0) | (rows >= n_rows) | (cols < 0) | (cols >= n_cols)
        if outside.any():
            k = int(np.argmax(outside))
            raise MatrixMarketError(f"index ({rows[k] + 1}, {cols[k] + 1}) outside {n_rows} x {n_cols}",
                                    path, entries[k][0])
    else:
        rows = np.empty(0, dtype=np.int64)
        cols = np.empty(0, dtype=np.int64)
        vals = np.empty(0)
    if symmetric:
        if n_rows != n_cols:
            raise MatrixMarketError("symmetric matrix must be square", path, size_lineno)
        strict = rows != cols  # mirror the stored triangle's off-diagonal entries
        rows, cols, vals = (np.concatenate([rows, cols[strict]]), np.concatenate([cols, rows[strict]]),
                            np.concatenate([vals, vals[strict]]))
    A = csr_from_coo(n_rows, n_cols, rows, cols, vals)
    name = path.rsplit("/", 1)[-1]
    name = name[:-4] if name.endswith(".mtx") else name
    return A, MatrixMetadata(name=name, n_rows=n_rows, n_cols=n_cols, nnz=A.nnz, symmetric=symmetric,
                             source=path)


def write_matrix_market(path: str, A: CsrMatrix, comment: str = "") -> None:
    """General real coordinate file, %.17g values (mmio.py:140-151): lossless round trip."""
    rows, cols, vals = A.to_coo()
    out = ["%%MatrixMarket matrix coordinate real general"]
    out += [f"% {ln}" for ln in comment.splitlines()] if comment else []
    out.append(f"{A.n_rows} {A.n_cols} {A.nnz}")
    out += [f"{r + 1} {c + 1} {v:.17g}" for r, c, v in zip(rows.tolist(), cols.tolist(), vals.tolist())]
    with open(path, "w", encoding="ascii") as fh:
        fh.write("\n".join(out) + "\n")
