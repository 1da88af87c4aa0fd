"""CSS-JSON descriptors: paper_2508_07879_b200.css_json against the
reference's reader / writer (proj/src/css_json.cpp:84-199, compiled into oracle/_ref when
json.hpp is available) and against the behaviour its tests pin
(proj/tests/test_css.cpp:195-258)."""
import json
import os

import numpy as np
import pytest

from paper_2508_07879_b200 import alist, codes, css_json

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "codes")


def _same_code(a, b):
    return (a.n == b.n and a.k == b.k and np.array_equal(a.hx.coo(), b.hx.coo())
            and np.array_equal(a.hz.coo(), b.hz.coo()))


def test_round_trips_inline_bb_and_files(tmp_path):
    """test_css.cpp:195-237: inline alists, bb parameters, external alist files."""
    code = codes.make_code("bb72")
    back = css_json.loads(css_json.dumps(code))
    assert _same_code(code, back) and back.name == "bb72" and back.d == 6
    l, m, a, b, k, d = codes.BUILTIN_SPECS["bb144"]
    c144 = codes.make_code("bb144")
    assert _same_code(c144, css_json.loads(css_json.dumps(c144, bb=(l, m, a, b))))
    (tmp_path / "hx.alist").write_text(alist.dumps(code.hx))
    (tmp_path / "hz.alist").write_text(alist.dumps(code.hz))
    (tmp_path / "code.json").write_text(css_json.dumps(code, "hx.alist", "hz.alist"))
    assert _same_code(code, css_json.load(str(tmp_path / "code.json")))


def test_committed_fixtures_load():
    assert _same_code(codes.make_code("bb72"), css_json.load(os.path.join(GOLD, "bb72_files.json")))
    assert _same_code(codes.make_code("bb144"), css_json.load(os.path.join(GOLD, "bb144_bb.json")))


def test_validation_messages():
    """test_css.cpp:239-258 and the loader's other diagnostics (css_json.cpp:18-150)."""
    code = codes.make_code("bb72")
    text = css_json.dumps(code)
    bad = text.replace('"k": 12', '"k": 11')
    assert bad != text
    with pytest.raises(css_json.CssJsonError, match="declared k=11 but rank computation gives k=12"):
        css_json.loads(bad)
    with pytest.raises(css_json.CssJsonError, match="declared n=73"):
        css_json.loads(text.replace('"n": 72', '"n": 73'))
    with pytest.raises(css_json.CssJsonError, match="invalid JSON"):
        css_json.loads("{not json")
    with pytest.raises(css_json.CssJsonError, match="css descriptor"):
        css_json.loads("{}")
    with pytest.raises(css_json.CssJsonError, match="cannot open css descriptor"):
        css_json.load("/nonexistent/code.json")
    doc = json.loads(text)
    for mutate, msg in (
            (lambda d: d.pop("params"), 'missing "params"'),
            (lambda d: d["params"].pop("n"), 'params is missing "n"'),
            (lambda d: d["params"].update(k=-1), "non-negative integer"),
            (lambda d: d.pop("construction"), 'missing "construction"'),
            (lambda d: d["construction"].update(bb={}), "not both or neither"),
            (lambda d: d["construction"].pop("alist_z"), 'string fields "alist_x" and "alist_z"'),
            (lambda d: d.update(construction={}), "not both or neither"),
            (lambda d: d.update(construction={"bb": {"l": 6, "m": 6, "a_terms": [[1]], "b_terms": []}}),
             "two-element"),
            (lambda d: d.update(construction={"bb": {"l": 6, "m": 6, "a_terms": 3}}), 'needs an array "a_terms"'),
            (lambda d: d.update(construction={"alist_x": "nope.alist", "alist_z": "nope.alist"}),
             "cannot open alist file")):
        d2 = json.loads(json.dumps(doc))
        mutate(d2)
        with pytest.raises(css_json.CssJsonError, match=msg):
            css_json.loads(json.dumps(d2))


def test_against_the_compiled_reference(ref):
    """The reference's own writer feeds our loader and vice versa; matrices, n, k, d agree."""
    if not ref.have_css_json():
        pytest.skip("oracle/_ref was built without css_json (json.hpp not found)")
    for name in ("bb72", "bb144"):
        rc = ref.code(name)
        ours = css_json.loads(ref.css_json_save(rc))
        mine = codes.make_code(name)
        assert _same_code(ours, mine) and ours.d == mine.d
        for text in (css_json.dumps(mine), css_json.dumps(mine, bb=codes.BUILTIN_SPECS[name][:4])):
            back = ref.css_json_load(text)
            assert (back.n, back.k, back.d) == (mine.n, mine.k, mine.d)
            assert np.array_equal(back.matrix_coo("hx"), mine.hx.coo())
            assert np.array_equal(back.matrix_coo("hz"), mine.hz.coo())
    bad = css_json.dumps(codes.make_code("bb72")).replace('"k": 12', '"k": 11')
    with pytest.raises(Exception, match="declared k=11 but rank computation gives k=12"):
        ref.css_json_load(bad)
    back = ref.css_json_load(open(os.path.join(GOLD, "bb72_files.json")).read(), GOLD)
    assert back.n == 72 and back.k == 12
