"""Host-side code model (paper_2508_07879_b200/codes.py, gf2.py) against the
reference: committed graph digests (tests/golden/graph_digests.json, produced
from the compiled reference), structural invariants the reference's tests pin
(proj/tests/test_css.cpp:44-57, :124-193) and the packed-vector KATs
(proj/tests/test_gf2.cpp:129-137)."""
import json
import os

import numpy as np
import pytest

from paper_2508_07879_b200 import codes, gf2

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("name", list(codes.BUILTIN_SPECS))
def test_graphs_match_reference_digests(name):
    with open(os.path.join(GOLDEN, "graph_digests.json")) as f:
        want = json.load(f)[name]
    code = codes.make_code(name)
    assert (code.n, code.k) == (want["n"], want["k"])
    assert code.graph_x.digest() == want["x"]
    assert code.graph_z.digest() == want["z"]
    assert code.combined_graph.digest() == want["combined"]


def test_registry_parameters():
    """proj/tests/test_css.cpp:124-170 + the [[784,24,24]] member."""
    want = {"bb72": (72, 12), "bb108": (108, 8), "bb144": (144, 12), "bb288": (288, 12),
            "bb756": (756, 16), "bb784": (784, 24)}
    for name, (n, k) in want.items():
        code = codes.make_code(name)
        assert (code.n, code.k) == (n, k)
        for g in (code.graph_x, code.graph_z):
            assert set(np.diff(g.check_offsets)) == {6} and set(np.diff(g.var_offsets)) == {3}


@pytest.mark.parametrize("name", ["bb72", "bb784"])
def test_graph_invariants(name):
    """var_edge_ids ascending, permutation, block-diagonal combined layout
    (proj/tests/test_css.cpp:44-57, :172-193)."""
    code = codes.make_code(name)
    g = code.combined_graph
    assert sorted(g.var_edges.tolist()) == list(range(g.num_edges))
    for n in range(g.num_vars):
        ids = g.var_edges[g.var_offsets[n]:g.var_offsets[n + 1]]
        assert (np.diff(ids.astype(np.int64)) > 0).all()
        assert (g.edge_var[ids] == n).all()
    mz, n_q = code.hz.rows, code.n
    top = g.edge_var[:g.check_offsets[mz]]
    bot = g.edge_var[g.check_offsets[mz]:]
    assert top.max() < n_q and bot.min() >= n_q
    assert np.array_equal(code.segments, [[0, mz, 0, n_q], [mz, mz + code.hx.rows, n_q, 2 * n_q]])


def test_toy_code_fixture():
    h = codes.toy_code_3x6()
    g = codes.build_tanner_graph(h)
    assert (g.num_checks, g.num_vars, g.num_edges) == (3, 6, 12)
    assert set(np.diff(g.check_offsets)) == {4} and set(np.diff(g.var_offsets)) == {2}
    assert codes.gf2_rank(h) == 2


def test_non_commuting_matrices_are_rejected():
    hx = codes.SparseMatrix.from_dense([[1, 1, 0]])
    hz = codes.SparseMatrix.from_dense([[1, 0, 0]])
    with pytest.raises(RuntimeError):
        codes.make_css_code("bad", hx, hz)


def test_packed_vector_layout_and_hex():
    bits = np.zeros(150, dtype=np.uint8)
    bits[[0, 63, 64, 149]] = 1
    w = gf2.pack_bits(bits)
    assert w.dtype == np.uint64 and w.shape == (3,)
    assert w[0] == (1 | (1 << 63)) and w[1] == 1 and w[2] == 1 << (149 - 128)
    assert np.array_equal(gf2.unpack_bits(w, 150), bits)

    def from01(s):
        return gf2.pack_bits(np.array([int(c) for c in s], dtype=np.uint8)), len(s)

    assert gf2.to_hex(*from01("1")) == "1"
    assert gf2.to_hex(*from01("0100")) == "2"
    assert gf2.to_hex(*from01("10110001")) == "d8"
    assert gf2.to_hex(*from01("11111")) == "f1"
    assert gf2.to_hex(np.zeros(1, dtype=np.uint64), 9) == "000"
    a, b = from01("1011"), from01("001")
    assert np.array_equal(gf2.unpack_bits(gf2.concat_bits(a[0], 4, b[0], 3), 7),
                          [1, 0, 1, 1, 0, 0, 1])


def test_syndrome_map_against_dense_product():
    code = codes.make_code("bb72")
    rng = np.random.default_rng(0)
    e = (rng.random((20, 72)) < 0.2).astype(np.uint8)
    assert np.array_equal(code.hz.mat_vec(e), (e @ code.hz.dense().T) & 1)


def test_extended_graph_has_identity_columns():
    code = codes.make_code("bb72")
    h, segs = codes.extended_graph(code)
    g = codes.build_tanner_graph(h)
    assert g.num_checks == 72 and g.num_vars == 2 * 72 + 72
    assert set(np.diff(g.check_offsets)) == {7}
    assert sorted(set(np.diff(g.var_offsets))) == [1, 3]
    assert segs.tolist() == [[0, 36, 0, 108], [36, 72, 108, 216]]
