"""CSS code descriptors (JSON) -> CssCode, the second on-disk format next to alist
(SURVEY.md §8f row 3).  Format, cross-checks and diagnostics follow the reference's loader
(proj/include/qldpc/css_json.hpp:9-32, proj/src/css_json.cpp:84-161):

    {"name": "bb72", "params": {"n": 72, "k": 12, "d": 6},
     "construction": {"bb": {"l": 6, "m": 6, "a_terms": [[3,0],[0,1],[0,2]],
                             "b_terms": [[0,3],[1,0],[2,0]]}}}

or, instead of "bb", {"alist_x": ..., "alist_z": ...} where a value containing a newline is
an inline alist payload and anything else a file path (relative paths resolve against
`base_dir`).  Loading REBUILDS the code and checks the declared n and k against the computed
ones; "d" is metadata.  Errors are CssJsonError (the reference throws std::runtime_error)."""
from __future__ import annotations

import json
import os
from typing import List, Optional, Sequence, Tuple

from . import alist
from .codes import CssCode, SparseMatrix, build_bb_code, make_css_code


class CssJsonError(RuntimeError):
    pass


def _count(node: dict, context: str, field: str) -> int:
    if field not in node:
        raise CssJsonError(f'css descriptor: {context} is missing "{field}"')
    v = node[field]
    if isinstance(v, bool) or not isinstance(v, int) or v < 0:
        raise CssJsonError(f'css descriptor: {context} field "{field}" must be a non-negative integer')
    return v


def _terms(node: dict, field: str) -> List[Tuple[int, int]]:
    if not isinstance(node.get(field), list):
        raise CssJsonError(f'css descriptor: bb construction needs an array "{field}"')
    out = []
    for entry in node[field]:
        ok = (isinstance(entry, list) and len(entry) == 2
              and all(isinstance(x, int) and not isinstance(x, bool) and x >= 0 for x in entry))
        if not ok:
            raise CssJsonError(f'css descriptor: each entry of "{field}" must be a two-element '
                               "[x_exp, y_exp] pair")
        out.append((entry[0], entry[1]))
    return out


def _alist_ref(value: str, base_dir: str) -> SparseMatrix:
    if "\n" in value:
        return alist.loads(value)
    path = value
    if not os.path.isabs(path) and base_dir:
        path = os.path.join(base_dir, path)
    try:
        return alist.load(path)
    except OSError:
        raise CssJsonError(f"cannot open alist file: {path}") from None


def loads(text: str, base_dir: str = "") -> CssCode:
    """reference: load_css_json (css_json.cpp:84-150)."""
    try:
        doc = json.loads(text)
    except ValueError as exc:
        raise CssJsonError(f"css descriptor: invalid JSON: {exc}") from None
    if not isinstance(doc, dict) or not isinstance(doc.get("name"), str):
        raise CssJsonError('css descriptor: top level must be an object with a string "name"')
    name = doc["name"]
    params = doc.get("params")
    if not isinstance(params, dict):
        raise CssJsonError('css descriptor: missing "params" object')
    declared_n = _count(params, "params", "n")
    declared_k = _count(params, "params", "k")
    declared_d = _count(params, "params", "d") if "d" in params else 0
    cons = doc.get("construction")
    if not isinstance(cons, dict):
        raise CssJsonError('css descriptor: missing "construction" object')
    has_bb = "bb" in cons
    has_alist = "alist_x" in cons or "alist_z" in cons
    if has_bb == has_alist:
        raise CssJsonError('css descriptor: construction must contain either "bb" or the '
                           '"alist_x"/"alist_z" pair, not both or neither')
    try:
        if has_bb:
            bb = cons["bb"]
            if not isinstance(bb, dict):
                raise CssJsonError('css descriptor: "bb" must be an object')
            code = build_bb_code(_count(bb, "bb construction", "l"), _count(bb, "bb construction", "m"),
                                 _terms(bb, "a_terms"), _terms(bb, "b_terms"), name, declared_d)
        else:
            if not isinstance(cons.get("alist_x"), str) or not isinstance(cons.get("alist_z"), str):
                raise CssJsonError('css descriptor: construction needs string fields "alist_x" and '
                                   '"alist_z"')
            code = make_css_code(name, _alist_ref(cons["alist_x"], base_dir),
                                 _alist_ref(cons["alist_z"], base_dir), declared_d)
    except ValueError as exc:  # builder argument errors (std::invalid_argument in the reference)
        raise CssJsonError(f"css descriptor '{name}': {exc}") from None
    if code.n != declared_n:
        raise CssJsonError(f"css descriptor '{name}': declared n={declared_n} but the construction "
                           f"has n={code.n}")
    if code.k != declared_k:
        raise CssJsonError(f"css descriptor '{name}': declared k={declared_k} but rank computation "
                           f"gives k={code.k}")
    return code


def load(path: str) -> CssCode:
    """reference: load_css_json_file (css_json.cpp:152-161)."""
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise CssJsonError(f"cannot open css descriptor: {path}") from None
    return loads(text, os.path.dirname(path))


def _params(code: CssCode) -> dict:
    out = {"n": code.n, "k": code.k}
    if code.d:
        out["d"] = code.d
    return out


def dumps(code: CssCode, alist_x_path: Optional[str] = None, alist_z_path: Optional[str] = None,
          bb: Optional[Tuple[int, int, Sequence[Tuple[int, int]], Sequence[Tuple[int, int]]]] = None) -> str:
    """reference: the three save_css_json overloads (css_json.cpp:163-199): inline alist
    payloads by default, external alist paths, or the bivariate-bicycle parameters
    (l, m, a_terms, b_terms)."""
    if bb is not None:
        l, m, a, b = bb
        cons = {"bb": {"l": l, "m": m, "a_terms": [list(t) for t in a], "b_terms": [list(t) for t in b]}}
    elif alist_x_path is not None or alist_z_path is not None:
        cons = {"alist_x": alist_x_path, "alist_z": alist_z_path}
    else:
        cons = {"alist_x": alist.dumps(code.hx), "alist_z": alist.dumps(code.hz)}
    return json.dumps({"name": code.name, "params": _params(code), "construction": cons}, indent=2) + "\n"
