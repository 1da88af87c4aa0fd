"""Pins the CPU oracle (oracle/msa_oracle.c) - the checker every GPU parity test
relies on - three ways, none of which needs a GPU:

1. the known-answer vectors the reference's own tests hold for this path
   (proj/tests/test_decoder.cpp:175-245, test_quantized.cpp:171-183),
2. golden fixtures produced by the UNMODIFIED compiled reference and committed
   under tests/golden/ (generator: tests/golden/make_golden.py),
3. a live differential against the compiled reference when oracle/_ref is
   present (always in the authoring container; prebuilt on the GPU box).
"""
import glob
import os
import types

import numpy as np
import pytest

from paper_2508_07879_b200 import DecoderConfig, codes, gf2
from tests.helpers import error_syndromes, random_ldpc_matrix, random_syndromes

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
MODES = ("float", "int8", "int16")


# ---- 1. known-answer vectors -----------------------------------------------------

def test_check_node_update_kats(oracle):
    q = [2.0, -3.0, 1.5]
    assert oracle.check_node_update(q, 0, 1.0).tolist() == [-1.5, 1.5, -2.0]
    assert oracle.check_node_update(q, 1, 1.0).tolist() == [1.5, -1.5, 2.0]
    assert oracle.check_node_update(q, 0, 0.5).tolist() == [-0.75, 0.75, -1.0]
    assert oracle.check_node_update([1.0] * 4, 0, 1.0).tolist() == [1.0] * 4
    r = oracle.check_node_update([0.0, -2.0], 0, 1.0)  # zero counts as positive
    assert r[0] == -2.0 and r[1] == 0.0
    assert oracle.check_node_update([5.0], 0, 0.8).tolist() == [0.8 * 64.0]
    assert oracle.check_node_update([5.0], 1, 0.8).tolist() == [-0.8 * 64.0]
    for bad in (([], 0, 1.0), (q, 0, 0.0), (q, 0, 1.5)):
        with pytest.raises(ValueError):
            oracle.check_node_update(*bad)


def test_variable_node_and_posterior_kats(oracle):
    assert oracle.variable_node_update(1.0, [-1.5, 2.0]).tolist() == [3.0, -0.5]
    assert oracle.variable_node_update(1.0, [7.0]).tolist() == [1.0]
    assert oracle.variable_node_update(0.0, [5.0, -5.0]).tolist() == [-5.0, 5.0]
    assert oracle.posterior_and_decision(1.0, [-1.5, 2.0]) == (1.5, 0)
    assert oracle.posterior_and_decision(1.0, [-3.0]) == (-2.0, 1)
    assert oracle.posterior_and_decision(1.0, [-1.0]) == (0.0, 0)  # exactly zero decides 0


def test_quantize_saturate_kats(oracle):
    cases = [(1.0, 8.0, 127, 8), (0.5, 256.0, 32767, 128), (100.0, 8.0, 127, 127),
             (-100.0, 8.0, 127, -127), (0.44, 8.0, 127, 4), (0.43, 8.0, 127, 3),
             (-0.4375, 8.0, 127, -4), (0.0, 8.0, 127, 0)]
    for v, sc, lim, want in cases:
        assert oracle.quantize_saturate(v, sc, lim) == want
    with pytest.raises(ValueError):
        oracle.quantize_saturate(float("nan"), 8.0, 127)


def test_two_minimum_trick_equals_definition(oracle):
    """proj/tests/test_decoder.cpp:207-221: a one-check graph decoded for one iteration
    yields exactly the definitional O(d^2) update, zeros and ties included."""
    rng = np.random.default_rng(17)
    for trial in range(200):
        deg = 2 + int(rng.integers(0, 6))
        q = rng.uniform(-4.0, 4.0, deg)
        if trial % 5 == 0:
            q[rng.integers(0, deg)] = 0.0
        if trial % 7 == 0:
            q[rng.integers(0, deg)] = q[-1]
        q32 = q.astype(np.float32)
        s_bit = int(rng.integers(0, 2))
        alpha = 1.0 if trial % 2 == 0 else 0.8
        want = oracle.check_node_update(q32.astype(np.float64), s_bit, alpha).astype(np.float32)
        # single check over `deg` variables, priors = q, zero VN effect after the CN stage:
        h = codes.SparseMatrix.from_rows(1, deg, [list(range(deg))])
        g = codes.build_tanner_graph(h)
        cfg = DecoderConfig(max_iterations=1, alpha=alpha, priors=q32.astype(np.float64).tolist())
        _, _, _, _, _, r = oracle.decode(g, cfg, gf2.pack_bits(np.array([s_bit], dtype=np.uint8)))
        assert np.array_equal(r.view(np.uint32), want.view(np.uint32))


def test_golden_node_ops_from_reference(oracle):
    z = np.load(os.path.join(GOLDEN, "node_ops.npz"))
    q = [2.0, -3.0, 1.5]
    assert np.array_equal(oracle.check_node_update(q, 0, 1.0), z["cn_a"])
    assert np.array_equal(oracle.check_node_update(q, 1, 1.0), z["cn_b"])
    assert np.array_equal(oracle.check_node_update(q, 0, 0.5), z["cn_c"])
    assert np.array_equal(oracle.check_node_update([0.0, -2.0], 0, 1.0), z["cn_zero"])
    assert oracle.check_node_update([5.0], 0, 0.8)[0] == z["cn_deg1"][0]
    assert np.array_equal(oracle.variable_node_update(1.0, [-1.5, 2.0]), z["vn_a"])
    assert np.array_equal(oracle.variable_node_update(1.0, [7.0]), z["vn_b"])


# ---- 2. golden fixtures from the compiled reference ---------------------------------

def _graph_from_npz(z):
    g = types.SimpleNamespace(num_checks=int(z["num_checks"]), num_vars=int(z["num_vars"]),
                              edge_var=z["edge_var"], check_offsets=z["check_offsets"],
                              var_offsets=z["var_offsets"], var_edges=z["var_edges"])
    return g


def _cfg_from_npz(z, mode):
    kw = {}
    for key in ("max_iterations", "alpha", "early_termination", "quant_scale", "priors"):
        if "cfg_" + key in z.files:
            v = z["cfg_" + key]
            kw[key] = v.tolist() if key == "priors" else v.item()
    if f"{mode}_quant_scale" in z.files and z[f"{mode}_quant_scale"].item():
        kw["quant_scale"] = float(z[f"{mode}_quant_scale"].item())
    kw.setdefault("early_termination", True)
    return DecoderConfig(arithmetic=mode, **kw)


GRAPH_FIXTURES = sorted(glob.glob(os.path.join(GOLDEN, "toy_*.npz")) +
                        glob.glob(os.path.join(GOLDEN, "irregular_*.npz")))
CSS_FIXTURES = sorted(glob.glob(os.path.join(GOLDEN, "css_*.npz")))


def test_golden_fixtures_exist():
    assert len(GRAPH_FIXTURES) >= 6 and len(CSS_FIXTURES) >= 4


@pytest.mark.parametrize("path", GRAPH_FIXTURES, ids=os.path.basename)
def test_oracle_matches_golden_graph_fixture(oracle, path):
    z = np.load(path)
    g = _graph_from_npz(z)
    for mode in MODES:
        if f"{mode}_estimate" not in z.files:
            continue
        cfg = _cfg_from_npz(z, mode)
        est, res, conv, its = oracle.decode_many(g, cfg, z["syndromes"], per_segment=False)
        assert np.array_equal(est, z[f"{mode}_estimate"]), (mode, "estimate")
        assert np.array_equal(res, z[f"{mode}_residual"]), (mode, "residual")
        assert np.array_equal(conv[:, 0], z[f"{mode}_converged"]), (mode, "converged")
        assert np.array_equal(its[:, 0], z[f"{mode}_iterations"]), (mode, "iterations")


@pytest.mark.parametrize("path", CSS_FIXTURES, ids=os.path.basename)
def test_oracle_matches_golden_css_fixture(oracle, path):
    z = np.load(path)
    name = os.path.basename(path).split("_")[1]
    code = codes.make_code(name)
    g = code.combined_graph
    # the committed syndromes are the reference sampler's: H * e must reproduce them
    ebits = np.concatenate([gf2.unpack_bits(z["ex"], code.n), gf2.unpack_bits(z["ez"], code.n)], 1)
    assert np.array_equal(gf2.unpack_bits(z["syndromes"], g.num_checks),
                          code.combined.mat_vec(ebits))
    for mode in MODES:
        cfg = DecoderConfig(max_iterations=int(z["max_iterations"]),
                            early_termination=bool(z["early"]), arithmetic=mode)
        est, res, conv, its = oracle.decode_many(g, cfg, z["syndromes"], code.segments)
        assert np.array_equal(est, z[f"{mode}_estimate"]), (mode, "estimate")
        assert np.array_equal(res, z[f"{mode}_residual"]), (mode, "residual")
        assert np.array_equal(conv, z[f"{mode}_conv_seg"]), (mode, "per-segment converged")
        assert np.array_equal(its, z[f"{mode}_iters_seg"]), (mode, "per-segment iterations")
        # decode_into view: AND / MAX over segments (decoder.cpp:204-213)
        assert np.array_equal(conv.all(axis=1), z[f"{mode}_converged"].astype(bool))
        assert np.array_equal(its.max(axis=1), z[f"{mode}_iterations"])


# ---- 3. live differential against the compiled reference ----------------------------

@pytest.mark.parametrize("mode", MODES)
def test_oracle_equals_compiled_reference_on_random_graphs(oracle, ref, mode):
    rng = np.random.default_rng(404)
    for round_ in range(8):
        h = random_ldpc_matrix(rng, 6 + int(rng.integers(0, 6)), 10 + int(rng.integers(0, 8)))
        g = codes.build_tanner_graph(h)
        rg = ref.graph_from_coo(h.rows, h.cols, h.coo())
        for k in ("edge_var", "edge_check", "check_offsets", "var_offsets", "var_edges"):
            assert np.array_equal(getattr(g, k), getattr(rg, k))
        priors = None
        if round_ % 2:
            priors = rng.uniform(0.3, 3.0, h.cols).tolist()
        for early in (True, False):
            cfg = DecoderConfig(max_iterations=10, early_termination=early, arithmetic=mode,
                                priors=priors, quant_scale=16.0 if priors else 0.0)
            syn = random_syndromes(rng, 12, h.rows, 0.3)
            rest, rres, rconv, rits = ref.decoder(rg, cfg).decode_many(syn)
            est, res, conv, its = oracle.decode_many(g, cfg, syn, per_segment=False)
            assert np.array_equal(est, rest) and np.array_equal(res, rres)
            assert np.array_equal(conv[:, 0], rconv) and np.array_equal(its[:, 0], rits)


def test_oracle_equals_compiled_reference_on_bb_codes(oracle, ref):
    rng = np.random.default_rng(5)
    for name in ("bb72", "bb144"):
        code = codes.make_code(name)
        rc = ref.code(name)
        _, _, syn = error_syndromes(code, rng, 40, 0.03)
        for mode in MODES:
            cfg = DecoderConfig(max_iterations=30, arithmetic=mode)
            rest, rres, rconv, rits = ref.decoder(rc, cfg).decode_many(syn)
            est, res, conv, its = oracle.decode_many(code.combined_graph, cfg, syn, code.segments,
                                                     per_segment=False)
            assert np.array_equal(est, rest) and np.array_equal(res, rres)
            assert np.array_equal(conv[:, 0], rconv) and np.array_equal(its[:, 0], rits)


def test_oracle_rejects_what_the_reference_rejects(oracle, ref):
    """decoder.cpp:373-387, :83-131."""
    g = codes.build_tanner_graph(codes.toy_code_3x6())
    rg = ref.toy_graph()
    bad_cfgs = [dict(alpha=0.0), dict(alpha=1.25), dict(max_iterations=0), dict(priors=[1.0, 2.0]),
                dict(priors=[1.0, 1.0, 1.0, float("inf"), 1.0, 1.0]),
                dict(arithmetic="int8", quant_scale=0.3), dict(arithmetic="int16", alpha=1e-6),
                dict(arithmetic="int8", quant_scale=-4.0)]
    for kw in bad_cfgs:
        cfg = DecoderConfig(**kw)
        assert not oracle.validate(g, cfg), kw
        with pytest.raises(ValueError):
            ref.decoder(rg, cfg)
    assert oracle.validate(g, DecoderConfig())


@pytest.mark.parametrize("mode,scale", [("float", 0.0), ("int8", 8.0), ("int16", 256.0)])
def test_per_shot_priors_oracle_equals_one_reference_decoder_per_shot(oracle, ref, mode, scale):
    """Soft syndromes (BASELINE config 5): the reference has priors per Decoder only
    (decoder.hpp:31-32), so the oracle's per-shot-prior entry point must equal one
    unmodified reference Decoder constructed per shot on the extended graph [H | I]."""
    from paper_2508_07879_b200 import DecoderConfig, codes, gf2
    code = codes.make_code("bb72")
    h, segs = codes.extended_graph(code)
    g = codes.build_tanner_graph(h)
    rng = np.random.default_rng(21)
    shots, n, mz, mx = 200, code.n, code.hz.rows, code.hx.rows
    meas = np.concatenate([np.arange(n, n + mz), np.arange(2 * n + mz, 2 * n + mz + mx)]).astype(np.uint32)
    err = (rng.random((shots, g.num_vars)) < 0.02).astype(np.uint8)
    syn = gf2.pack_bits(h.mat_vec(err))
    soft = np.abs(1.0 + 0.6 * rng.standard_normal((shots, meas.size))) * 5.0 + 0.2
    if mode != "float":
        soft = np.maximum(np.round(soft * scale), 1.0) / scale
    cfg = DecoderConfig(max_iterations=25, arithmetic=mode, quant_scale=scale,
                        priors=[4.0] * g.num_vars)
    oe, ores, oc, oi = oracle.decode_many_soft(g, cfg, syn, meas, soft, None, per_segment=False)
    rg = ref.graph_from_coo(h.rows, h.cols, h.coo())
    re_, rres, rc, ri = ref.decode_many_soft(rg, cfg, syn, meas, soft)
    assert np.array_equal(oe, re_) and np.array_equal(ores, rres)
    assert np.array_equal(oc[:, 0], rc) and np.array_equal(oi[:, 0], ri)
    # and the per-shot values matter: a constant prior gives different outcomes
    fe, _, _, _ = oracle.decode_many(g, cfg, syn, None, per_segment=False)
    assert not np.array_equal(fe, oe)


@pytest.mark.parametrize("mode", ["float", "int8", "int16"])
def test_oracle_matches_golden_soft_fixture(oracle, mode):
    """tests/golden/soft_bb144_p0.01.npz: soft syndromes on diag([Hz | I], [Hx | I]), every
    shot decoded by its own unmodified reference Decoder (priors per Decoder,
    decoder.hpp:31-32) - the oracle's per-shot-prior entry point reproduces it."""
    from paper_2508_07879_b200 import DecoderConfig, codes
    d = np.load(os.path.join(GOLDEN, "soft_bb144_p0.01.npz"))
    code = codes.make_code(str(d["code"]))
    h, _ = codes.extended_graph(code)
    g = codes.build_tanner_graph(h)
    stored = d[f"{mode}_soft"].astype(np.float64)
    if mode != "float":
        stored = stored / (8.0 if mode == "int8" else 256.0)
    cfg = DecoderConfig(max_iterations=int(d["max_iterations"]), arithmetic=mode,
                        priors=[float(d["prior_data"])] * g.num_vars)
    est, res, conv, its = oracle.decode_many_soft(g, cfg, d["syndromes"], d["soft_vars"], stored,
                                                  None, per_segment=False)
    assert np.array_equal(est, d[f"{mode}_estimate"]) and np.array_equal(res, d[f"{mode}_residual"])
    assert np.array_equal(conv[:, 0], d[f"{mode}_converged"])
    assert np.array_equal(its[:, 0], d[f"{mode}_iterations"])
    assert 0 < d[f"{mode}_converged"].mean() and d[f"{mode}_iterations"].max() > 3
