"""Host-side code model used to FEED the decoder: parity-check matrices, the
Tanner-graph edge tables the C-ABI consumes, and the bivariate-bicycle family.

This is cold, run-once host code (out of scope for
kernels).  It exists because the GPU box has no reference tree: tests and
bench build their graphs here, and tests/test_codes.py pins every array
against the reference's `build_tanner_graph` / `build_bb_code`
(proj/src/tanner_graph.cpp:7-41, proj/src/css_code.cpp:14-49, :122-138) and
against committed golden digests.
"""
from __future__ import annotations

import dataclasses
import hashlib
from typing import Dict, List, Sequence, Tuple

import numpy as np


@dataclasses.dataclass(frozen=True)
class TannerGraph:
    """reference: struct TannerGraph (proj/include/qldpc/tanner_graph.hpp:15-48).

    Edges are numbered check-major (row by row, columns ascending); `var_edges`
    lists each variable's edge ids in ascending order.
    """

    num_checks: int
    num_vars: int
    edge_var: np.ndarray       # uint32 [E]
    edge_check: np.ndarray     # uint32 [E]
    check_offsets: np.ndarray  # uint32 [M + 1]
    var_offsets: np.ndarray    # uint32 [N + 1]
    var_edges: np.ndarray      # uint32 [E]

    @property
    def num_edges(self) -> int:
        return int(self.edge_var.shape[0])

    def digest(self) -> str:
        h = hashlib.sha256()
        h.update(np.array([self.num_checks, self.num_vars, self.num_edges], dtype="<u8").tobytes())
        for arr in (self.edge_var, self.edge_check, self.check_offsets, self.var_offsets,
                    self.var_edges):
            h.update(np.ascontiguousarray(arr, dtype="<u4").tobytes())
        return h.hexdigest()


@dataclasses.dataclass(frozen=True)
class SparseMatrix:
    """Binary matrix as sorted per-row column supports."""

    rows: int
    cols: int
    row_support: Tuple[Tuple[int, ...], ...]

    @staticmethod
    def from_rows(rows: int, cols: int, supports: Sequence[Sequence[int]]) -> "SparseMatrix":
        if len(supports) != rows:
            raise ValueError("one support list per row required")
        out = []
        for r, sup in enumerate(supports):
            s = sorted(int(c) for c in sup)
            if any(c < 0 or c >= cols for c in s):
                raise ValueError(f"row {r}: column out of range")
            if any(a == b for a, b in zip(s, s[1:])):
                raise ValueError(f"row {r}: duplicate entry")
            out.append(tuple(s))
        return SparseMatrix(rows, cols, tuple(out))

    @staticmethod
    def from_dense(dense: Sequence[Sequence[int]]) -> "SparseMatrix":
        d = np.asarray(dense)
        return SparseMatrix.from_rows(d.shape[0], d.shape[1],
                                      [np.flatnonzero(row).tolist() for row in d])

    @property
    def nnz(self) -> int:
        return sum(len(s) for s in self.row_support)

    def transpose(self) -> "SparseMatrix":
        cols: List[List[int]] = [[] for _ in range(self.cols)]
        for r, sup in enumerate(self.row_support):
            for c in sup:
                cols[c].append(r)
        return SparseMatrix.from_rows(self.cols, self.rows, cols)

    def dense(self) -> np.ndarray:
        d = np.zeros((self.rows, self.cols), dtype=np.uint8)
        for r, sup in enumerate(self.row_support):
            d[r, list(sup)] = 1
        return d

    def coo(self) -> np.ndarray:
        """(nnz, 2) uint32 array of (row, col), row-major."""
        out = [(r, c) for r, sup in enumerate(self.row_support) for c in sup]
        return np.asarray(out, dtype=np.uint32).reshape(-1, 2)

    def mat_vec(self, v_bits: np.ndarray) -> np.ndarray:
        """Syndrome map s_m = XOR of v over row m's support (proj/src/gf2.cpp:215-228).
        v_bits: (..., cols) uint8 -> (..., rows) uint8."""
        v_bits = np.asarray(v_bits, dtype=np.uint8)
        out = np.zeros(v_bits.shape[:-1] + (self.rows,), dtype=np.uint8)
        for r, sup in enumerate(self.row_support):
            if sup:
                out[..., r] = np.bitwise_xor.reduce(v_bits[..., list(sup)], axis=-1)
        return out


def hstack(a: SparseMatrix, b: SparseMatrix) -> SparseMatrix:
    return SparseMatrix.from_rows(
        a.rows, a.cols + b.cols,
        [list(ra) + [c + a.cols for c in rb] for ra, rb in zip(a.row_support, b.row_support)])


def block_diag(top: SparseMatrix, bottom: SparseMatrix) -> SparseMatrix:
    rows = [list(r) for r in top.row_support]
    rows += [[c + top.cols for c in r] for r in bottom.row_support]
    return SparseMatrix.from_rows(top.rows + bottom.rows, top.cols + bottom.cols, rows)


def gf2_rank(m: SparseMatrix) -> int:
    """GF(2) rank by elimination on bit-packed rows (Python ints as bitsets)."""
    rows = []
    for sup in m.row_support:
        x = 0
        for c in sup:
            x |= 1 << c
        rows.append(x)
    rank = 0
    basis: Dict[int, int] = {}
    for x in rows:
        while x:
            top = x.bit_length() - 1
            if top in basis:
                x ^= basis[top]
            else:
                basis[top] = x
                rank += 1
                break
    return rank


def build_tanner_graph(h: SparseMatrix) -> TannerGraph:
    if h.rows == 0 or h.cols == 0 or h.nnz == 0:
        raise ValueError("build_tanner_graph: matrix must have rows, columns and a nonzero")
    edge_var = np.fromiter((c for sup in h.row_support for c in sup), dtype=np.uint32)
    deg = np.fromiter((len(s) for s in h.row_support), dtype=np.int64, count=h.rows)
    check_offsets = np.zeros(h.rows + 1, dtype=np.uint32)
    check_offsets[1:] = np.cumsum(deg)
    edge_check = np.repeat(np.arange(h.rows, dtype=np.uint32), deg)
    # stable sort by variable keeps edge ids ascending within each variable
    var_edges = np.argsort(edge_var, kind="stable").astype(np.uint32)
    vdeg = np.bincount(edge_var, minlength=h.cols)
    var_offsets = np.zeros(h.cols + 1, dtype=np.uint32)
    var_offsets[1:] = np.cumsum(vdeg)
    return TannerGraph(h.rows, h.cols, edge_var, edge_check, check_offsets, var_offsets, var_edges)


@dataclasses.dataclass(frozen=True)
class CssCode:
    """reference: class CssCode (proj/include/qldpc/css_code.hpp:44-79).  X errors
    are seen through hz (graph_x), Z errors through hx (graph_z); the combined
    graph is diag(hz, hx) with syndrome s_x ++ s_z and estimate e_x ++ e_z."""

    name: str
    hx: SparseMatrix
    hz: SparseMatrix
    n: int
    k: int
    d: int
    graph_x: TannerGraph
    graph_z: TannerGraph
    combined: SparseMatrix
    combined_graph: TannerGraph

    @property
    def segments(self) -> np.ndarray:
        """(2, 4) uint32: (check_begin, check_end, var_begin, var_end) for X then Z
        (proj/src/decoder.cpp:415-424)."""
        mz, mx, n = self.hz.rows, self.hx.rows, self.n
        return np.asarray([[0, mz, 0, n], [mz, mz + mx, n, 2 * n]], dtype=np.uint32)


def make_css_code(name: str, hx: SparseMatrix, hz: SparseMatrix, d: int = 0) -> CssCode:
    if hx.rows == 0 or hz.rows == 0 or hx.cols == 0:
        raise ValueError("parity-check matrices must be non-empty")
    if hx.cols != hz.cols:
        raise ValueError("hx and hz must have the same number of columns")
    prod = (hx.dense().astype(np.int64) @ hz.dense().astype(np.int64).T) & 1
    if prod.any():
        i, j = np.argwhere(prod)[0]
        raise RuntimeError(f"stabilizers do not commute: hx row {i} / hz row {j}")
    n = hx.cols
    k = n - gf2_rank(hx) - gf2_rank(hz)
    combined = block_diag(hz, hx)
    return CssCode(name, hx, hz, n, k, d, build_tanner_graph(hz), build_tanner_graph(hx),
                   combined, build_tanner_graph(combined))


def _monomial_sum(l: int, m: int, terms: Sequence[Tuple[int, int]]) -> SparseMatrix:
    red = [(a % l, b % m) for a, b in terms]
    if len(set(red)) != len(red):
        raise ValueError("duplicate monomial after exponent reduction")
    rows = []
    for u in range(l):
        for v in range(m):
            rows.append([((u + a) % l) * m + (v + b) % m for a, b in red])
    return SparseMatrix.from_rows(l * m, l * m, rows)


def build_bb_code(l: int, m: int, a_terms: Sequence[Tuple[int, int]],
                  b_terms: Sequence[Tuple[int, int]], name: str = "", d: int = 0) -> CssCode:
    """Bivariate bicycle code: H_X = [A | B], H_Z = [B^T | A^T]
    (proj/include/qldpc/css_code.hpp:28-41)."""
    if l <= 0 or m <= 0 or not a_terms or not b_terms:
        raise ValueError("build_bb_code: l, m positive and term lists non-empty")
    a = _monomial_sum(l, m, a_terms)
    b = _monomial_sum(l, m, b_terms)
    hx = hstack(a, b)
    hz = hstack(b.transpose(), a.transpose())
    return make_css_code(name or f"bb{2 * l * m}", hx, hz, d)


# name -> (l, m, A terms, B terms, k, d).  bb72..bb756 are the reference's registry
# (proj/src/css_code.cpp:145-162); bb784 is the [[784,24,24]] code of BASELINE.json,
# constructible through the same builder.
BUILTIN_SPECS = {
    "bb72": (6, 6, [(3, 0), (0, 1), (0, 2)], [(0, 3), (1, 0), (2, 0)], 12, 6),
    "bb108": (9, 6, [(3, 0), (0, 1), (0, 2)], [(0, 3), (1, 0), (2, 0)], 8, 10),
    "bb144": (12, 6, [(3, 0), (0, 1), (0, 2)], [(0, 3), (1, 0), (2, 0)], 12, 12),
    "bb288": (12, 12, [(3, 0), (0, 2), (0, 7)], [(0, 3), (1, 0), (2, 0)], 12, 18),
    "bb756": (21, 18, [(3, 0), (0, 10), (0, 17)], [(0, 5), (3, 0), (19, 0)], 16, 34),
    "bb784": (28, 14, [(26, 0), (0, 6), (0, 8)], [(0, 7), (9, 0), (20, 0)], 24, 24),
}

_CODE_CACHE: Dict[str, CssCode] = {}


def make_code(name: str) -> CssCode:
    if name not in BUILTIN_SPECS:
        raise ValueError(f"unknown code '{name}' (available: {', '.join(BUILTIN_SPECS)})")
    if name not in _CODE_CACHE:
        l, m, a, b, k, d = BUILTIN_SPECS[name]
        code = build_bb_code(l, m, a, b, name, d)
        if code.k != k:
            raise RuntimeError(f"{name}: construction yields k={code.k}, expected {k}")
        _CODE_CACHE[name] = code
    return _CODE_CACHE[name]


def toy_code_3x6() -> SparseMatrix:
    """reference fixture (proj/src/css_code.cpp:185-189)."""
    return SparseMatrix.from_dense([[1, 0, 1, 1, 0, 1], [1, 1, 0, 1, 1, 0], [0, 1, 1, 0, 1, 1]])


def extended_graph(code: CssCode) -> Tuple[SparseMatrix, np.ndarray]:
    """Phenomenological-noise extension diag([Hz | I], [Hx | I]): one extra
    degree-1 variable per check models a flipped measurement.
    Returns the matrix and its (2, 4) segment table."""
    mz, mx, n = code.hz.rows, code.hx.rows, code.n
    top = hstack(code.hz, SparseMatrix.from_rows(mz, mz, [[i] for i in range(mz)]))
    bot = hstack(code.hx, SparseMatrix.from_rows(mx, mx, [[i] for i in range(mx)]))
    segs = np.asarray([[0, mz, 0, n + mz], [mz, mz + mx, n + mz, 2 * n + mz + mx]],
                      dtype=np.uint32)
    return block_diag(top, bot), segs
