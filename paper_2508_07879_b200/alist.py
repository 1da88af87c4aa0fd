"""alist interchange format -> SparseMatrix, so user-supplied (non-BB, irregular)
parity-check matrices can be fed to the decoder.  Format and
error behaviour follow the reference's loader (proj/include/qldpc/alist.hpp:10-27,
proj/src/alist.cpp:48-131): 1-based indices, zero padding accepted, column and row
support blocks cross-checked, diagnostics carry the offending line number."""
from __future__ import annotations

from typing import List

from .codes import SparseMatrix


class AlistError(RuntimeError):
    """Malformed alist input (the reference throws std::runtime_error, alist.cpp:36-39)."""


def _ints(lines: List[str], idx: int, what: str) -> List[int]:
    if idx >= len(lines):
        raise AlistError(f"alist: line {idx + 1}: unexpected end of input while reading {what}")
    try:
        return [int(tok) for tok in lines[idx].split()]
    except ValueError:
        raise AlistError(f"alist: line {idx + 1}: non-integer token in {what}") from None


def loads(text: str) -> SparseMatrix:
    lines = [ln for ln in text.splitlines() if ln.strip()]  # blank lines are skipped (alist.cpp:18-31)
    head = _ints(lines, 0, "dimensions")
    if len(head) != 2 or head[0] <= 0 or head[1] <= 0:
        raise AlistError("alist: line 1: expected positive 'N M'")
    n, m = head
    degs = _ints(lines, 1, "maximum degrees")
    if len(degs) != 2:
        raise AlistError("alist: line 2: expected two maximum degrees")
    col_deg = _ints(lines, 2, "column degrees")
    row_deg = _ints(lines, 3, "row degrees")
    if len(col_deg) != n:
        raise AlistError(f"alist: line 3: expected {n} column degrees, found {len(col_deg)}")
    if len(row_deg) != m:
        raise AlistError(f"alist: line 4: expected {m} row degrees, found {len(row_deg)}")
    if max(col_deg) > degs[0] or max(row_deg) > degs[1]:
        raise AlistError("alist: line 2: a listed degree exceeds the declared maximum")
    cols: List[List[int]] = []
    for c in range(n):
        ln = 4 + c
        entries = [v for v in _ints(lines, ln, f"support of column {c + 1}") if v != 0]
        if len(entries) != col_deg[c]:
            raise AlistError(f"alist: line {ln + 1}: column {c + 1} lists {len(entries)} entries "
                             f"but its degree is {col_deg[c]}")
        if any(v < 1 or v > m for v in entries):
            raise AlistError(f"alist: line {ln + 1}: row index out of range")
        cols.append(sorted(v - 1 for v in entries))
    rows: List[List[int]] = []
    for r in range(m):
        ln = 4 + n + r
        entries = [v for v in _ints(lines, ln, f"support of row {r + 1}") if v != 0]
        if len(entries) != row_deg[r]:
            raise AlistError(f"alist: line {ln + 1}: row {r + 1} lists {len(entries)} entries "
                             f"but its degree is {row_deg[r]}")
        if any(v < 1 or v > n for v in entries):
            raise AlistError(f"alist: line {ln + 1}: column index out of range")
        rows.append(sorted(v - 1 for v in entries))
    if len(lines) > 4 + n + m and any(ln.strip() for ln in lines[4 + n + m:]):
        raise AlistError(f"alist: line {4 + n + m + 1}: trailing content")
    from_cols = [[] for _ in range(m)]
    for c, sup in enumerate(cols):
        for r in sup:
            from_cols[r].append(c)
    for r in range(m):
        if sorted(from_cols[r]) != rows[r]:
            raise AlistError(f"alist: line {4 + n + r + 1}: row {r + 1} disagrees with the "
                             "column supports")
    return SparseMatrix.from_rows(m, n, rows)


def load(path: str) -> SparseMatrix:
    with open(path) as f:
        return loads(f.read())


def dumps(h: SparseMatrix) -> str:
    """Canonical form (unpadded, single spaces, one list per line): loads(dumps(h)) == h."""
    cols = h.transpose().row_support
    out = [f"{h.cols} {h.rows}",
           f"{max(len(c) for c in cols)} {max(len(r) for r in h.row_support)}",
           " ".join(str(len(c)) for c in cols), " ".join(str(len(r)) for r in h.row_support)]
    out += [" ".join(str(v + 1) for v in c) for c in cols]
    out += [" ".join(str(v + 1) for v in r) for r in h.row_support]
    return "\n".join(out) + "\n"
