"""GPU parity tests proper: the CUDA path (through the C-ABI) against the CPU
oracle and — where the prebuilt library travelled — the compiled reference, on
identical graphs, priors and syndromes.  Bit-exact for every mode the reference
has (float, int8, int16); structure follows proj/tests/test_decoder.cpp and
proj/tests/test_quantized.cpp.
"""
import numpy as np
import pytest

from paper_2508_07879_b200 import (Decoder, DecoderConfig, codes, decode, decode_batch,
                                   decode_css, gf2)
from tests.helpers import (error_syndromes, random_ldpc_matrix, random_regular63_matrix, random_syndrome,
                           random_syndromes)

pytestmark = pytest.mark.gpu

REF_MODES = ("float", "int8", "int16")


def assert_matches_oracle(oracle, graph, cfg, syndromes, segments=None, dec=None, messages=False):
    """CUDA (single-shot path) == oracle on every syndrome: estimate, residual,
    per-segment converged and iterations; optionally the edge messages."""
    own = dec is None
    dec = dec or Decoder(graph, cfg, segments=segments)
    try:
        for s in syndromes:
            oe, ores, oc, oi, oq, orr = oracle.decode(graph, cfg, s, segments)
            if messages:
                e, r, c, i, q, rr = dec.decode_debug(s)
            else:
                e, r, c, i = dec.decode_segments(s)
            assert np.array_equal(e, oe), "estimate differs"
            assert np.array_equal(r, ores), "residual differs"
            assert np.array_equal(c, oc), "converged differs"
            assert np.array_equal(i, oi), "iterations differ"
            if messages:
                # q is defined by the last VN stage in both; r likewise by the last CN stage
                assert np.array_equal(q.view(np.uint32) if q.dtype == np.float32 else q,
                                      oq.view(np.uint32) if oq.dtype == np.float32 else oq), "q differs"
                assert np.array_equal(rr.view(np.uint32) if rr.dtype == np.float32 else rr,
                                      orr.view(np.uint32) if orr.dtype == np.float32 else orr), "r differs"
    finally:
        if own:
            dec.close()


def test_device_is_blackwell(gpu_lib):
    assert gpu_lib["cc"][0] >= 10, gpu_lib
    assert gpu_lib["sms"] > 0


@pytest.mark.parametrize("mode", REF_MODES + ("half",))
def test_zero_syndrome_is_a_one_iteration_fixed_point(mode):
    """proj/tests/test_decoder.cpp:247-267, test_quantized.cpp:206-220."""
    for name in ("bb72", "bb108", "bb144", "bb288", "bb756", "bb784"):
        code = codes.make_code(name)
        g = code.combined_graph
        zero = np.zeros(gf2.num_words(g.num_checks), dtype=np.uint64)
        cfg = DecoderConfig(arithmetic=mode)
        out = decode(g, zero, cfg)
        assert out.converged and out.iterations_used == 1
        assert not out.error_estimate.any() and not out.syndrome_residual.any()
        cfg.early_termination = False
        out = decode(g, zero, cfg)
        assert out.converged and out.iterations_used == cfg.max_iterations
        assert not out.error_estimate.any()


@pytest.mark.parametrize("mode", REF_MODES)
def test_toy_code_every_syndrome(oracle, mode):
    """proj/tests/test_decoder.cpp:269-294 and :417-424: converged iff s == 0,
    iterations 1 or 10 (period-2 oscillation), and bit-exact with the oracle
    including every edge message."""
    h = codes.toy_code_3x6()
    g = codes.build_tanner_graph(h)
    cfg = DecoderConfig(alpha=0.8, max_iterations=10, arithmetic=mode)
    syndromes = [gf2.pack_bits(np.array([(mask >> m) & 1 for m in range(3)], dtype=np.uint8))
                 for mask in range(8)]
    with Decoder(g, cfg) as dec:
        for mask, s in enumerate(syndromes):
            out = dec.decode(s)
            est_bits = gf2.unpack_bits(out.error_estimate, 6)
            hs = h.mat_vec(est_bits)
            assert np.array_equal(gf2.unpack_bits(out.syndrome_residual, 3),
                                  hs ^ gf2.unpack_bits(s, 3))
            if mode == "float":
                assert out.converged == (mask == 0)
                assert out.iterations_used == (1 if mask == 0 else 10)
        assert_matches_oracle(oracle, g, cfg, syndromes, dec=dec, messages=True)


@pytest.mark.parametrize("mode", REF_MODES)
def test_bb72_x_graph_matches_oracle_bit_for_bit(oracle, mode):
    """proj/tests/test_decoder.cpp:426-434 / test_quantized.cpp:250-258."""
    code = codes.make_code("bb72")
    rng = np.random.default_rng(71)
    for trial in range(25):
        cfg = DecoderConfig(alpha=0.8, max_iterations=10, early_termination=trial % 2 == 0,
                            arithmetic=mode)
        s = random_syndrome(rng, code.hz.rows, 0.1)
        assert_matches_oracle(oracle, code.graph_x, cfg, [s], messages=True)


@pytest.mark.parametrize("mode", REF_MODES)
def test_irregular_graphs_with_unit_degrees(oracle, mode):
    """proj/tests/test_decoder.cpp:436-447: degree-1 checks and variables."""
    rng = np.random.default_rng(5)
    for _ in range(10):
        h = random_ldpc_matrix(rng, 6 + int(rng.integers(0, 6)), 10 + int(rng.integers(0, 8)))
        g = codes.build_tanner_graph(h)
        for trial in range(10):
            cfg = DecoderConfig(alpha=0.8, max_iterations=10, early_termination=trial % 2 == 0,
                                arithmetic=mode)
            s = random_syndrome(rng, g.num_checks, 0.3)
            assert_matches_oracle(oracle, g, cfg, [s], messages=True)


def test_non_uniform_priors(oracle):
    """proj/tests/test_decoder.cpp:449-458."""
    g = codes.build_tanner_graph(codes.toy_code_3x6())
    cfg = DecoderConfig(alpha=0.8, max_iterations=10, priors=[0.5, 1.25, 2.0, 0.75, 3.0, 1.5])
    syndromes = [gf2.pack_bits(np.array([(mask >> m) & 1 for m in range(3)], dtype=np.uint8))
                 for mask in range(8)]
    assert_matches_oracle(oracle, g, cfg, syndromes, messages=True)
    # negative and zero priors take the same code path in the reference
    cfg.priors = [-0.5, 0.0, 2.0, -0.75, 3.0, 1e-3]
    assert_matches_oracle(oracle, g, cfg, syndromes, messages=True)


@pytest.mark.parametrize("mode", ("int8", "int16"))
def test_saturating_priors(oracle, mode):
    """proj/tests/test_quantized.cpp:272-283."""
    g = codes.build_tanner_graph(codes.toy_code_3x6())
    cfg = DecoderConfig(alpha=0.8, max_iterations=10, arithmetic=mode, quant_scale=16.0,
                        priors=[20.0, 1.0, -2.0, 500.0, 0.25, 1.0])
    syndromes = [gf2.pack_bits(np.array([(mask >> m) & 1 for m in range(3)], dtype=np.uint8))
                 for mask in range(8)]
    assert_matches_oracle(oracle, g, cfg, syndromes, messages=True)


def test_validation_errors():
    """proj/tests/test_decoder.cpp:296-326, test_quantized.cpp:185-204."""
    g = codes.build_tanner_graph(codes.toy_code_3x6())
    for bad in (dict(alpha=0.0), dict(alpha=1.25), dict(max_iterations=0),
                dict(priors=[1.0, 2.0]),
                dict(priors=[1.0, 1.0, 1.0, float("inf"), 1.0, 1.0]),
                dict(arithmetic="int8", quant_scale=0.3),
                dict(arithmetic="int16", alpha=1e-6),
                dict(arithmetic="int8", quant_scale=-4.0)):
        with pytest.raises(ValueError):
            Decoder(g, DecoderConfig(**bad))
    with pytest.raises(ValueError, match="quantizes to 0"):
        Decoder(g, DecoderConfig(arithmetic="int8", quant_scale=0.3))
    code = codes.make_code("bb72")
    with Decoder(code.graph_x, DecoderConfig()) as dec:
        with pytest.raises(ValueError):
            dec.decode(np.zeros(1, dtype=np.uint64), bits=35)
        with pytest.raises(ValueError):
            dec.decode_css_into(np.zeros(1, dtype=np.uint64), np.zeros(1, dtype=np.uint64))
    with pytest.raises(ValueError):
        decode(code.graph_x, np.zeros(2, dtype=np.uint64), DecoderConfig(), bits=72)


def test_zero_shot_and_null_buffer_batches_through_the_c_abi():
    """decode_batch on an empty span returns an empty result before any work
    (proj/src/decoder.cpp:617); through the C-ABI that is QB_OK with no launch, while
    a non-empty batch with a NULL buffer is rejected as an invalid argument."""
    code = codes.make_code("bb72")
    for mode in ("float", "int8"):
        with Decoder(code, DecoderConfig(arithmetic=mode)) as dec:
            before = dec.launch_count()
            est, res, conv, its = dec.decode_batch_segments(np.zeros((0, 2), dtype=np.uint64))
            assert est.shape == (0, 3) and res.shape == (0, 2)
            assert conv.shape == (0, 2) and its.shape == (0, 2)
            dec.decode_batch_raw(0, 0, 0, None, 0, 0)
            assert dec.launch_count() == before
            with pytest.raises(ValueError, match="NULL"):
                dec.decode_batch_raw(4, 0, 0, None, 0, 0)
            # the handle is still usable after the rejected call
            out = dec.decode(np.zeros(2, dtype=np.uint64))
            assert out.converged and out.iterations_used == 1


def test_decoder_instances_are_reusable():
    """proj/tests/test_decoder.cpp:328-339."""
    code = codes.make_code("bb72")
    rng = np.random.default_rng(3)
    with Decoder(code.graph_x, DecoderConfig()) as dec:
        s = random_syndrome(rng, code.hz.rows, 0.1)
        first = dec.decode(s)
        dec.decode(random_syndrome(rng, code.hz.rows, 0.4))
        again = dec.decode(s)
        assert first.same_as(again)


@pytest.mark.parametrize("mode", REF_MODES)
def test_batch_equals_sequential_map(oracle, mode):
    """proj/tests/test_decoder.cpp:341-377, test_quantized.cpp:285-301."""
    code = codes.make_code("bb72")
    cfg = DecoderConfig(alpha=0.8, arithmetic=mode)
    rng = np.random.default_rng(29)
    syndromes = [random_syndrome(rng, code.hz.rows, 0.08) for _ in range(64)]
    batch = decode_batch(code.graph_x, syndromes, cfg, 1)
    assert len(batch) == 64
    with Decoder(code.graph_x, cfg) as dec:
        for s, b in zip(syndromes, batch):
            assert b.same_as(dec.decode(s))
    for workers in (2, 8):
        again = decode_batch(code.graph_x, syndromes, cfg, workers)
        assert all(a.same_as(b) for a, b in zip(again, batch))
    assert decode_batch(code.graph_x, [], cfg, 4) == []
    bad = list(syndromes)
    bad[7] = np.zeros(1, dtype=np.uint64)
    with pytest.raises(ValueError):
        decode_batch(code.graph_x, bad, cfg, 2, bits=[36] * 7 + [5] + [36] * 56)
    oe, ores, oc, oi = oracle.decode_many(code.graph_x, cfg, np.stack(syndromes))
    for k, b in enumerate(batch):
        assert np.array_equal(b.error_estimate, oe[k]) and b.iterations_used == oi[k, 0]
        assert b.converged == bool(oc[k, 0]) and np.array_equal(b.syndrome_residual, ores[k])


@pytest.mark.parametrize("mode", REF_MODES)
def test_combined_decode_equals_two_separate_decodes(mode):
    """proj/tests/test_decoder.cpp:379-405, test_quantized.cpp:303-320."""
    for name in ("bb72", "bb144"):
        code = codes.make_code(name)
        rng = np.random.default_rng(59)
        for trial in range(24):
            cfg = DecoderConfig(alpha=0.8, early_termination=trial % 2 == 0, arithmetic=mode)
            s_x = random_syndrome(rng, code.hz.rows, 0.06)
            s_z = random_syndrome(rng, code.hx.rows, 0.06)
            cx, cz = decode_css(code, s_x, s_z, cfg)
            assert cx.same_as(decode(code.graph_x, s_x, cfg))
            assert cz.same_as(decode(code.graph_z, s_z, cfg))


@pytest.mark.parametrize("name,mode", [("bb144", "float"), ("bb144", "int8"), ("bb784", "float"),
                                       ("bb784", "int8"), ("bb784", "int16"), ("bb756", "float")])
def test_css_batch_matches_oracle(oracle, name, mode):
    """Combined-graph decode of error-derived syndromes (the bench / campaign
    workload, proj/src/bench.cpp:203-211) at several error rates, batch path,
    bit-exact with the oracle per segment."""
    code = codes.make_code(name)
    rng = np.random.default_rng(2024)
    for p, iters, early in ((0.01, 50, True), (0.03, 30, True), (0.02, 10, False)):
        cfg = DecoderConfig(max_iterations=iters, early_termination=early, arithmetic=mode)
        _, _, syn = error_syndromes(code, rng, 96, p)
        with Decoder(code, cfg) as dec:
            est, res, conv, its = dec.decode_batch_segments(syn)
            # and the single-shot path agrees with the batch path
            e1, r1, c1, i1 = dec.decode_segments(syn[5])
        oe, ores, oc, oi = oracle.decode_many(code.combined_graph, cfg, syn, code.segments)
        assert np.array_equal(est, oe)
        assert np.array_equal(res, ores)
        assert np.array_equal(conv, oc)
        assert np.array_equal(its, oi)
        assert np.array_equal(e1, oe[5]) and np.array_equal(r1, ores[5])
        assert np.array_equal(c1, oc[5]) and np.array_equal(i1, oi[5])


def test_against_compiled_reference(ref):
    """The unmodified reference Decoder (prebuilt oracle/_ref) on its own bench
    pool recipe: decode_into and decode_css_into outcomes equal ours exactly."""
    for name in ("bb144", "bb784"):
        rc = ref.code(name)
        code = codes.make_code(name)
        pool = ref.syndrome_pool(rc, 0.02, 1, 128)
        for mode in REF_MODES:
            cfg = DecoderConfig(max_iterations=50, arithmetic=mode)
            rest, rres, rconv, rits = ref.decoder(rc, cfg).decode_many(pool)
            with Decoder(code, cfg) as dec:
                est, res, conv, its = dec.decode_batch_segments(pool)
            assert np.array_equal(est, rest)
            assert np.array_equal(res, rres)
            assert np.array_equal(conv.all(axis=1), rconv.astype(bool))
            assert np.array_equal(its.max(axis=1), rits)


def test_large_batch_soundness_properties():
    """Size-independent properties at scale (proj/tests/acceptance.cpp:56-100):
    residual == H*e_hat ^ s for every shot, converged <=> residual == 0,
    iterations within [1, cap], and the batch is reproducible."""
    code = codes.make_code("bb784")
    rng = np.random.default_rng(7)
    shots = 20000
    _, _, syn = error_syndromes(code, rng, shots, 0.02)
    cfg = DecoderConfig(max_iterations=30)
    with Decoder(code, cfg) as dec:
        est, res, conv, its = dec.decode_batch_segments(syn)
        est2, res2, conv2, its2 = dec.decode_batch_segments(syn)
    assert np.array_equal(est, est2) and np.array_equal(res, res2)
    assert np.array_equal(conv, conv2) and np.array_equal(its, its2)
    g = code.combined_graph
    e_bits = gf2.unpack_bits(est, g.num_vars)
    s_bits = gf2.unpack_bits(syn, g.num_checks)
    hs = code.combined.mat_vec(e_bits)
    assert np.array_equal(gf2.unpack_bits(res, g.num_checks), hs ^ s_bits)
    mz = code.hz.rows
    rb = gf2.unpack_bits(res, g.num_checks)
    assert np.array_equal(conv[:, 0].astype(bool), ~rb[:, :mz].any(axis=1))
    assert np.array_equal(conv[:, 1].astype(bool), ~rb[:, mz:].any(axis=1))
    assert its.min() >= 1 and its.max() <= 30
    assert conv.mean() > 0.9


# ---- every kernel variant must produce the same bits -----------------------------------

OPT_KERNEL, OPT_LATENCY_IO, OPT_LATENCY_SHAPE, OPT_GROUP_THREADS = 0, 1, 2, 3
OPT_BATCH_CTAS, OPT_BATCH_NPT, OPT_LATENCY_NPT, OPT_FAST_PATH, OPT_BATCH_SHAPE = 4, 5, 6, 7, 8
INFO_BATCH_REGULAR, INFO_LATENCY_CLUSTER, INFO_LATENCY_LEAN = 104, 103, 106


@pytest.mark.parametrize("mode", REF_MODES)
@pytest.mark.parametrize("name", ["bb72", "bb144", "bb784"])
def test_regular_and_cluster_kernels_match_oracle(oracle, name, mode):
    """(6,3)-regular fast path: the thread-block-cluster single-shot kernel (CTA rank =
    segment) in both nodes-per-thread classes, the one-CTA-per-shot shape (generic CSR
    kernel), and every variant of the batch kernel, against the oracle bit for bit
    (messages included on the single-shot path)."""
    code = codes.make_code(name)
    g = code.combined_graph
    rng = np.random.default_rng(11)
    _, _, syn = error_syndromes(code, rng, 48, 0.03)
    for iters, early in ((12, True), (7, False)):
        cfg = DecoderConfig(max_iterations=iters, early_termination=early, arithmetic=mode)
        oe, ores, oc, oi = oracle.decode_many(g, cfg, syn, code.segments)
        with Decoder(code, cfg) as dec:
            assert dec.get_option(INFO_BATCH_REGULAR) == 1
            for shape in (1, 2):
                dec.set_option(OPT_LATENCY_SHAPE, shape)
                assert dec.get_option(INFO_LATENCY_CLUSTER) == (1 if shape == 2 else 0)
                for npt in (1, 2, 3):
                    dec.set_option(OPT_LATENCY_NPT, npt)
                    assert_matches_oracle(oracle, g, cfg, syn[:6], code.segments, dec=dec,
                                          messages=True)
            # lean cluster kernel: every way of delivering the syndrome, incl. the
            # persistent doorbell (no launch per shot)
            dec.set_option(OPT_LATENCY_SHAPE, 0)
            dec.set_option(OPT_LATENCY_NPT, 0)
            assert dec.get_option(INFO_LATENCY_LEAN) == 1
            for io_mode in (0, 1, 2):
                dec.set_option(OPT_LATENCY_IO, io_mode)
                launches = dec.launch_count()
                assert_matches_oracle(oracle, g, cfg, syn[:12], code.segments, dec=dec)
                if io_mode == 2:
                    assert dec.launch_count() - launches <= 2, "doorbell mode must not launch per shot"
            dec.set_option(OPT_LATENCY_IO, 0)
            for bshape in (1, 2):  # CTA per shot / CTA per (shot, segment) work item
                dec.set_option(OPT_BATCH_SHAPE, bshape)
                assert dec.get_option(OPT_BATCH_SHAPE) == bshape
                for npt in ((0,) if bshape == 1 else (1, 2, 3, 4, 6, 8, 11)):
                    dec.set_option(OPT_BATCH_NPT, npt)
                    for fast in (1, 0):
                        dec.set_option(OPT_FAST_PATH, fast)
                        est, res, conv, its = dec.decode_batch_segments(syn)
                        assert np.array_equal(est, oe) and np.array_equal(res, ores), (npt, "bits")
                        assert np.array_equal(conv, oc) and np.array_equal(its, oi), (npt, "flags")
                        est2, _, conv2, its2 = dec.decode_batch_segments(syn, want_residual=False)
                        assert np.array_equal(est2, oe) and np.array_equal(its2, oi)
            dec.set_option(OPT_KERNEL, 1)  # generic CSR kernel on the same handle
            assert dec.get_option(INFO_BATCH_REGULAR) == 0
            est, res, conv, its = dec.decode_batch_segments(syn)
            assert np.array_equal(est, oe) and np.array_equal(its, oi)


def test_regular_kernel_is_rejected_on_irregular_graphs():
    g = codes.build_tanner_graph(codes.toy_code_3x6())
    with Decoder(g, DecoderConfig()) as dec:
        assert dec.get_option(INFO_BATCH_REGULAR) == 0
        with pytest.raises(ValueError):
            dec.set_option(OPT_KERNEL, 2)


def test_half_mode_tracks_float_decisions():
    """fp16 messages have no reference counterpart (decoder.hpp:16): they must
    agree with the fp32 decoder on the overwhelming majority of shots and never
    claim convergence with a wrong syndrome."""
    code = codes.make_code("bb144")
    rng = np.random.default_rng(3)
    _, _, syn = error_syndromes(code, rng, 2000, 0.01)
    with Decoder(code, DecoderConfig(max_iterations=50)) as d32, \
            Decoder(code, DecoderConfig(max_iterations=50, arithmetic="half")) as d16:
        e32, r32, c32, i32 = d32.decode_batch_segments(syn)
        e16, r16, c16, i16 = d16.decode_batch_segments(syn)
    g = code.combined_graph
    hs = code.combined.mat_vec(gf2.unpack_bits(e16, g.num_vars))
    assert np.array_equal(gf2.unpack_bits(r16, g.num_checks), hs ^ gf2.unpack_bits(syn, g.num_checks))
    agree = (e32 == e16).all(axis=1).mean()
    assert agree > 0.98, agree
    assert abs(c32.mean() - c16.mean()) < 0.01


OPT_HALF_PAIRS = 10


@pytest.mark.parametrize("name,shots,p", [("bb72", 257, 0.03), ("bb144", 1001, 0.02),
                                          ("bb784", 600, 0.01)])
def test_half_mode_every_kernel_gives_identical_results(name, shots, p):
    """Half mode is fp16 arithmetic in every kernel, so the packed two-shots-per-
    thread batch kernel, the one-shot-per-thread batch variants, the generic CSR
    kernel and the single-shot cluster kernel must agree bit for bit (odd shot
    counts exercise the half-empty last pair)."""
    code = codes.make_code(name)
    rng = np.random.default_rng(17)
    _, _, syn = error_syndromes(code, rng, shots, p)
    g = code.combined_graph
    priors = (0.5 + rng.random(g.num_vars) * 4.0).tolist()
    for cfg in (DecoderConfig(max_iterations=30, arithmetic="half"),
                DecoderConfig(max_iterations=7, early_termination=False, arithmetic="half"),
                DecoderConfig(max_iterations=30, arithmetic="half", priors=priors)):
        with Decoder(code, cfg) as dec:
            assert dec.get_option(OPT_HALF_PAIRS) == 1
            want = dec.decode_batch_segments(syn)
            hs = code.combined.mat_vec(gf2.unpack_bits(want[0], g.num_vars))
            assert np.array_equal(gf2.unpack_bits(want[1], g.num_checks),
                                  hs ^ gf2.unpack_bits(syn, g.num_checks))
            for variant in (1, 2, 3, 4, 6, 8):
                try:
                    dec.set_option(OPT_BATCH_NPT, variant)
                except ValueError:
                    continue  # CTA shape does not fit this code
                got = dec.decode_batch_segments(syn)
                assert all(np.array_equal(a, b) for a, b in zip(got, want)), variant
            dec.set_option(OPT_BATCH_NPT, 0)
            dec.set_option(OPT_HALF_PAIRS, 0)
            assert dec.get_option(OPT_HALF_PAIRS) == 0
            got = dec.decode_batch_segments(syn)
            assert all(np.array_equal(a, b) for a, b in zip(got, want)), "unpaired"
            for k in range(0, shots, max(1, shots // 40)):
                one = dec.decode_segments(syn[k])
                assert all(np.array_equal(a, b[k]) for a, b in zip(one, want)), k
            dec.set_option(OPT_KERNEL, 1)
            got = dec.decode_batch_segments(syn)
            assert all(np.array_equal(a, b) for a, b in zip(got, want)), "generic"


@pytest.mark.parametrize("name,shots,p", [("bb72", 257, 0.03), ("bb144", 1001, 0.02),
                                          ("bb784", 601, 0.01), ("bb784", 300, 0.04)])
def test_int8_on_the_packed_fp16_kernel_is_bit_exact(oracle, name, shots, p):
    """int8 batches run two shots per thread on packed fp16 instructions (int8
    quantities are exact fp16 integers, Q16 scaling as one fused multiply-add,
    kernel_lean_h2.cuh).  Must equal the integer oracle (decoder.cpp:260-283) bit
    for bit - uniform and per-variable priors incl. saturating and negative ones,
    several alphas / scales, odd shot counts - and the one-shot-per-thread kernel."""
    code = codes.make_code(name)
    rng = np.random.default_rng(23)
    _, _, syn = error_syndromes(code, rng, shots, p)
    g = code.combined_graph
    priors = (rng.uniform(0.2, 20.0, g.num_vars) * rng.choice([-1.0, 1.0], g.num_vars, p=[0.05, 0.95]))
    cfgs = [DecoderConfig(max_iterations=30, arithmetic="int8"),
            DecoderConfig(max_iterations=7, early_termination=False, arithmetic="int8"),
            DecoderConfig(max_iterations=30, arithmetic="int8", priors=priors.tolist()),
            DecoderConfig(max_iterations=20, arithmetic="int8", alpha=0.625, quant_scale=20.0),
            DecoderConfig(max_iterations=20, arithmetic="int8", alpha=1.0, quant_scale=100.0),
            DecoderConfig(max_iterations=20, arithmetic="int8", alpha=0.3, quant_scale=3.0,
                          priors=(-priors).tolist())]
    paired = 0
    for cfg in cfgs:
        oe, ores, oc, oi = oracle.decode_many(g, cfg, syn, code.segments)
        with Decoder(code, cfg) as dec:
            paired += dec.get_option(OPT_HALF_PAIRS)
            got = dec.decode_batch_segments(syn)
            assert np.array_equal(got[0], oe) and np.array_equal(got[1], ores), "bits"
            assert np.array_equal(got[2], oc) and np.array_equal(got[3], oi), "flags"
            dec.set_option(OPT_HALF_PAIRS, 0)
            assert dec.get_option(OPT_HALF_PAIRS) == 0
            got = dec.decode_batch_segments(syn)
            assert np.array_equal(got[0], oe) and np.array_equal(got[3], oi), "unpaired"
    assert paired >= 4, "the packed kernel was not selected"


@pytest.mark.parametrize("mode", ["float", "int16", "int8"])
def test_tma_tiles_ragged_tail_and_unaligned_buffers(oracle, mode):
    """The lean batch kernels (one shot per thread: float / int16; two shots per thread on
    packed fp16 instructions: int8) stream syndromes in tiles of up to 16 shots (one TMA bulk
    copy per tile).  20001 shots leave a ragged last tile (odd row count -> plain loads), and a
    buffer that starts on an odd 104-byte row is only 8-byte aligned (every tile -> plain
    loads): both must give the same results as the aligned bulk copies and the oracle."""
    import torch
    code = codes.make_code("bb784")
    g = code.combined_graph
    shots = 20001
    rng = np.random.default_rng(99)
    _, _, syn = error_syndromes(code, rng, shots, 0.01)
    cfg = DecoderConfig(max_iterations=20, arithmetic=mode)
    sw, ew = gf2.num_words(g.num_checks), gf2.num_words(g.num_vars)
    host = torch.from_numpy(syn.view(np.int64).copy())
    d_all = torch.zeros((shots + 1, sw), dtype=torch.int64, device="cuda")
    d_all[1:] = host.cuda()
    d_aligned = d_all[1:].clone()
    assert d_aligned.data_ptr() % 16 == 0 and d_all[1:].data_ptr() % 16 == 8
    outs = []
    stream = torch.cuda.current_stream().cuda_stream
    with Decoder(code, cfg) as dec:
        for d_syn in (d_aligned, d_all[1:]):
            d_est = torch.full((shots, ew), -1, dtype=torch.int64, device="cuda")
            d_res = torch.full((shots, sw), -1, dtype=torch.int64, device="cuda")
            d_conv = torch.zeros((shots, 2), dtype=torch.uint8, device="cuda")
            d_its = torch.zeros((shots, 2), dtype=torch.int32, device="cuda")
            dec.decode_batch_device(shots, d_syn.data_ptr(), d_est.data_ptr(), d_res.data_ptr(),
                                    d_conv.data_ptr(), d_its.data_ptr(), stream)
            torch.cuda.synchronize()
            outs.append((d_est.cpu().numpy().view(np.uint64), d_res.cpu().numpy().view(np.uint64),
                         d_conv.cpu().numpy(), d_its.cpu().numpy().astype(np.uint32)))
    assert all(np.array_equal(a, b) for a, b in zip(outs[0], outs[1])), "aligned vs unaligned"
    # every tile size gives the same bits (QB_OPT_BATCH_TILE = 13)
    with Decoder(code, cfg) as dec:
        for tile in (1, 2, 5, 16):
            dec.set_option(13, tile)
            d_est = torch.full((shots, ew), -1, dtype=torch.int64, device="cuda")
            d_conv = torch.zeros((shots, 2), dtype=torch.uint8, device="cuda")
            d_its = torch.zeros((shots, 2), dtype=torch.int32, device="cuda")
            dec.decode_batch_device(shots, d_aligned.data_ptr(), d_est.data_ptr(), None,
                                    d_conv.data_ptr(), d_its.data_ptr(), stream)
            torch.cuda.synchronize()
            assert np.array_equal(d_est.cpu().numpy().view(np.uint64), outs[0][0]), tile
            assert np.array_equal(d_its.cpu().numpy().astype(np.uint32), outs[0][3]), tile
    for sl in (slice(0, 200), slice(shots - 200, shots)):
        oe, ores, oc, oi = oracle.decode_many(g, cfg, syn[sl], code.segments)
        assert np.array_equal(outs[0][0][sl], oe) and np.array_equal(outs[0][1][sl], ores)
        assert np.array_equal(outs[0][2][sl], oc) and np.array_equal(outs[0][3][sl], oi)
    # every shot: residual == H e_hat xor s, converged <=> zero residual (size-independent)
    est = gf2.unpack_bits(outs[0][0], g.num_vars)
    res = gf2.unpack_bits(outs[0][1], g.num_checks)
    assert np.array_equal(res, code.combined.mat_vec(est) ^ gf2.unpack_bits(syn, g.num_checks))
    mz = code.hz.rows
    assert np.array_equal(outs[0][2][:, 0] == 1, ~res[:, :mz].any(axis=1))
    assert np.array_equal(outs[0][2][:, 1] == 1, ~res[:, mz:].any(axis=1))
    # the other batch kernels on pre-filled (-1) output buffers: padding bits of the packed
    # rows must come back as zeros from every one of them
    n2 = 2001
    with Decoder(code, cfg) as dec:
        for opt, val in ((OPT_BATCH_SHAPE, 1), (OPT_KERNEL, 1)):
            dec.set_option(opt, val)
            d_est = torch.full((n2, ew), -1, dtype=torch.int64, device="cuda")
            d_res = torch.full((n2, sw), -1, dtype=torch.int64, device="cuda")
            d_conv = torch.zeros((n2, 2), dtype=torch.uint8, device="cuda")
            d_its = torch.zeros((n2, 2), dtype=torch.int32, device="cuda")
            dec.decode_batch_device(n2, d_aligned.data_ptr(), d_est.data_ptr(), d_res.data_ptr(),
                                    d_conv.data_ptr(), d_its.data_ptr(), stream)
            torch.cuda.synchronize()
            assert np.array_equal(d_est.cpu().numpy().view(np.uint64), outs[0][0][:n2]), (opt, val)
            assert np.array_equal(d_res.cpu().numpy().view(np.uint64), outs[0][1][:n2]), (opt, val)


def test_memcpy_protocol_graph_and_event_timing(oracle):
    """Single shots through the paper's protocol (H2D copy, kernel, D2H copy): as one
    CUDA-graph launch (default) and as three stream operations, results identical to the
    oracle; with QB_OPT_LATENCY_EVENTS the CUDA-event span of the protocol is reported."""
    OPT_LATENCY_EVENTS, OPT_LATENCY_GRAPH, INFO_LAST_EVENT_NS = 11, 12, 108
    code = codes.make_code("bb784")
    g = code.combined_graph
    rng = np.random.default_rng(4)
    _, _, syn = error_syndromes(code, rng, 40, 0.02)
    cfg = DecoderConfig(max_iterations=10, early_termination=False)
    with Decoder(code, cfg) as dec:
        dec.set_option(OPT_LATENCY_IO, 1)
        for graph in (1, 0, 1):
            dec.set_option(OPT_LATENCY_GRAPH, graph)
            assert dec.get_option(OPT_LATENCY_GRAPH) == graph
            launches = dec.launch_count()
            assert_matches_oracle(oracle, g, cfg, syn, code.segments, dec=dec)
            assert dec.launch_count() - launches == len(syn)
        dec.set_option(OPT_LATENCY_EVENTS, 1)
        wall, ev, _ = dec.latency_run(syn.view(np.uint64), 5, 50)
        assert dec.get_option(INFO_LAST_EVENT_NS) > 0
        # device span of copy + kernel + copy: above the kernel alone, below the host wall clock
        assert 2_000 < np.median(ev) <= np.median(wall) < 1_000_000
        dec.set_option(OPT_LATENCY_EVENTS, 0)
        _, kern, _ = dec.latency_run(syn.view(np.uint64), 5, 50)
        assert np.median(kern) < np.median(ev)
        # QB_OPT_LATENCY_WAIT = 1: completion read off the copied record's tags instead of a
        # stream synchronize - same results, graph or not, also when interleaved with the
        # other single-shot protocols and with batch calls on the same handle
        want = oracle.decode_many(g, cfg, syn, code.segments)
        dec.set_option(18, 1)
        assert dec.get_option(18) == 1
        for graph in (1, 0):
            dec.set_option(OPT_LATENCY_GRAPH, graph)
            assert_matches_oracle(oracle, g, cfg, syn, code.segments, dec=dec)
        for k, io_mode in enumerate((1, 0, 1, 2, 1, 1, 0, 2, 1)):
            dec.set_option(OPT_LATENCY_IO, io_mode)
            got = dec.decode_segments(syn[k])
            assert all(np.array_equal(a, b[k]) for a, b in zip(got, want)), (k, io_mode)
            if k == 4:
                batch = dec.decode_batch_segments(syn)
                assert all(np.array_equal(a, b) for a, b in zip(batch, want))
        with pytest.raises(ValueError):
            dec.set_option(18, 2)


# ---- per-edge messages of the THROUGHPUT kernels ----------------------------------------

def _bits(a):
    return a.view(np.uint32) if a.dtype == np.float32 else a


@pytest.mark.parametrize("mode", REF_MODES)
@pytest.mark.parametrize("p", [0.01, 0.03])
def test_batch_kernel_messages_match_oracle_bitwise(oracle, mode, p):
    """north star: "per-edge messages within 1e-5 relative" - checked where the time is
    spent: the persistent batch kernels (decode_lean_kernel for float / int16,
    decode_lean_h2_kernel for int8) decoding a whole bb784 batch with syndrome tiles, work
    queues and the first-iteration-from-the-syndrome shortcut ACTIVE, dump the final q and r
    of selected shots; they equal the oracle's (reference semantics
    proj/src/decoder.cpp:245-335) bit for bit, which is stronger than the stated tolerance.
    Every syndrome appears twice in a row so that, on the two-shots-per-thread kernel, both
    lanes of a pair stop together."""
    code = codes.make_code("bb784")
    g = code.combined_graph
    rng = np.random.default_rng(31)
    _, _, syn1 = error_syndromes(code, rng, 96, p)
    syn = np.repeat(syn1, 2, axis=0)
    for cfg in (DecoderConfig(max_iterations=50, arithmetic=mode),
                DecoderConfig(max_iterations=10, early_termination=False, arithmetic=mode)):
        oe, ores, oc, oi = oracle.decode_many(g, cfg, syn1, code.segments)
        # shots covering the spread of iteration counts, incl. one-iteration segments (r is
        # implicit there) and non-converged ones
        order = np.argsort(oi.max(axis=1), kind="stable")
        picks = sorted({int(order[0]), int(order[len(order) // 3]), int(order[len(order) // 2]),
                        int(order[-2]), int(order[-1])})
        if cfg.early_termination:
            assert oi.min() == 1, "the sample must contain one-iteration segments"
        with Decoder(code, cfg) as dec:
            assert dec.get_option(104) == 1
            for k in picks:
                for lane in ((0, 1) if k == picks[0] else (k & 1,)):
                    est, res, conv, its, q, r = dec.decode_batch_debug(syn, 2 * k + lane)
                    assert np.array_equal(est[::2], oe) and np.array_equal(est[1::2], oe)
                    assert np.array_equal(its[::2], oi) and np.array_equal(conv[1::2], oc)
                    _, _, _, _, oq, orr = oracle.decode(g, cfg, syn1[k], code.segments)
                    assert np.array_equal(_bits(q), _bits(oq)), ("q", k, oi[k])
                    assert np.array_equal(_bits(r), _bits(orr)), ("r", k, oi[k])


def test_batch_kernel_messages_half_mode_equal_the_single_shot_kernel():
    """fp16 messages have no oracle; the packed batch kernel's messages must equal the
    single-shot half kernel's (same arithmetic, lane by lane)."""
    code = codes.make_code("bb144")
    rng = np.random.default_rng(32)
    _, _, syn1 = error_syndromes(code, rng, 40, 0.03)
    syn = np.repeat(syn1, 2, axis=0)
    cfg = DecoderConfig(max_iterations=30, arithmetic="half")
    with Decoder(code, cfg) as dec:
        for k in (0, 7, 21, 39):
            est, res, conv, its, q, r = dec.decode_batch_debug(syn, 2 * k + 1)
            e1, r1, c1, i1, q1, rr1 = dec.decode_debug(syn1[k])
            assert np.array_equal(est[2 * k], e1) and np.array_equal(its[2 * k + 1], i1)
            assert np.array_equal(_bits(q), _bits(q1)) and np.array_equal(_bits(r), _bits(rr1))


@pytest.mark.parametrize("mode", REF_MODES)
def test_degree_padded_batch_kernel_messages_match_oracle_bitwise(oracle, mode):
    """The same for decode_ell_kernel / decode_ell_h2_kernel on the extended graph
    diag([Hz | I], [Hx | I]) of BASELINE config 5 (absorbed measurement variables included:
    their q stays the prior, decoder.cpp:324-329)."""
    code = codes.make_code("bb144")
    h, segs = codes.extended_graph(code)
    g = codes.build_tanner_graph(h)
    rng = np.random.default_rng(33)
    err = (rng.random((48, g.num_vars)) < 0.02).astype(np.uint8)
    syn1 = gf2.pack_bits(h.mat_vec(err))
    syn = np.repeat(syn1, 2, axis=0)
    cfg = DecoderConfig(max_iterations=30, arithmetic=mode, priors=[3.9] * g.num_vars)
    oe, ores, oc, oi = oracle.decode_many(g, cfg, syn1, segs)
    with Decoder(g, cfg, segments=segs) as dec:
        assert dec.get_option(107) == 703
        for k in (0, 11, 30, 47):
            est, res, conv, its, q, r = dec.decode_batch_debug(syn, 2 * k)
            assert np.array_equal(est[::2], oe) and np.array_equal(its[1::2], oi)
            _, _, _, _, oq, orr = oracle.decode(g, cfg, syn1[k], segs)
            assert np.array_equal(_bits(q), _bits(oq)), ("q", k)
            assert np.array_equal(_bits(r), _bits(orr)), ("r", k)


@pytest.mark.parametrize("mode", REF_MODES)
def test_annealed_slot_permutation_leaves_results_unchanged(oracle, mode):
    """QB_OPT_SLOT_SPREAD = 2 (slot permutation refined by simulated annealing) only moves
    messages inside their check's block: outcomes and per-edge messages of the batch kernels
    stay those of the oracle."""
    code = codes.make_code("bb144")
    g = code.combined_graph
    rng = np.random.default_rng(77)
    _, _, syn1 = error_syndromes(code, rng, 64, 0.03)
    syn = np.repeat(syn1, 2, axis=0)
    cfg = DecoderConfig(max_iterations=30, arithmetic=mode)
    oe, ores, oc, oi = oracle.decode_many(g, cfg, syn1, code.segments)
    with Decoder(code, cfg) as dec:
        dec.set_option(14, 2)
        assert dec.get_option(14) == 2
        for k in (0, 17, 63):
            est, res, conv, its, q, r = dec.decode_batch_debug(syn, 2 * k + 1)
            assert np.array_equal(est[::2], oe) and np.array_equal(res[1::2], ores)
            assert np.array_equal(its[::2], oi) and np.array_equal(conv[1::2], oc)
            _, _, _, _, oq, orr = oracle.decode(g, cfg, syn1[k], code.segments)
            assert np.array_equal(_bits(q), _bits(oq)) and np.array_equal(_bits(r), _bits(orr))
        with pytest.raises(ValueError):
            dec.set_option(14, 3)


@pytest.mark.parametrize("l,m,lean", [(32, 30, True), (31, 32, False)])
def test_largest_segments_of_the_regular_kernels_and_the_first_size_beyond(oracle, l, m, lean):
    """Maximum sizes: 960 checks per segment is the largest graph the (6,3)-regular item and
    cluster kernels take (message blocks of one segment in one CTA's shared memory, syndrome
    in the kernel parameters); one size up (992) the generic CSR kernel must take over.  Both
    decode a batch and single shots exactly as the oracle, float and int8."""
    code = codes.build_bb_code(l, m, [(3, 0), (0, 1), (0, 2)], [(0, 3), (1, 0), (2, 0)], f"bb{2 * l * m}")
    g = code.combined_graph
    assert g.num_checks == 2 * l * m
    rng = np.random.default_rng(l * m)
    _, _, syn = error_syndromes(code, rng, 40, 0.01)
    for mode in ("float", "int8"):
        cfg = DecoderConfig(max_iterations=20, arithmetic=mode)
        oe, ores, oc, oi = oracle.decode_many(g, cfg, syn, code.segments)
        with Decoder(code, cfg) as dec:
            assert dec.get_option(INFO_BATCH_REGULAR) == (1 if lean else 0)
            assert dec.get_option(INFO_LATENCY_LEAN) == (1 if lean else 0)
            est, res, conv, its = dec.decode_batch_segments(syn)
            assert np.array_equal(est, oe) and np.array_equal(res, ores)
            assert np.array_equal(conv, oc) and np.array_equal(its, oi)
            for io_mode in ((0, 1, 2) if lean else (0, 1)):
                dec.set_option(OPT_LATENCY_IO, io_mode)
                for k in (0, 13, 39):
                    e1, r1, c1, i1 = dec.decode_segments(syn[k])
                    assert np.array_equal(e1, oe[k]) and np.array_equal(r1, ores[k])
                    assert np.array_equal(c1, oc[k]) and np.array_equal(i1, oi[k])
    assert oi.max() > 2 and oc.min() in (0, 1)


@pytest.mark.parametrize("mode", REF_MODES)
def test_unstructured_regular_graphs_on_the_regular_kernels(oracle, mode):
    """The (6,3)-regular kernels assume the degrees, not the bivariate-bicycle structure: random
    regular graphs (one segment, and two different graphs as two segments of unequal size) go
    through the item kernel, its slot permutation and the cluster kernel, and decode as the
    oracle does - outcomes and, for one shot of the batch, every edge message."""
    rng = np.random.default_rng(20260824)
    h1 = random_regular63_matrix(rng, 100)
    h2 = random_regular63_matrix(rng, 61)
    both = codes.block_diag(h1, h2)
    cases = [(h1, None), (both, np.array([[0, 100, 0, 200], [100, 161, 200, 322]], dtype=np.uint32))]
    for h, segs in cases:
        g = codes.build_tanner_graph(h)
        err = (rng.random((33, g.num_vars)) < 0.03).astype(np.uint8)
        syn1 = gf2.pack_bits(h.mat_vec(err))
        syn = np.repeat(syn1, 2, axis=0)  # both lanes of a packed pair stop together
        for iters, early in ((25, True), (6, False)):
            cfg = DecoderConfig(max_iterations=iters, early_termination=early, arithmetic=mode)
            oe, ores, oc, oi = oracle.decode_many(g, cfg, syn1, segs)
            with Decoder(g, cfg, segments=segs) as dec:
                assert dec.get_option(INFO_BATCH_REGULAR) == 1 and dec.get_option(INFO_LATENCY_LEAN) == 1
                for spread in (0, 1, 2):
                    dec.set_option(14, spread)
                    est, res, conv, its, q, r = dec.decode_batch_debug(syn, 2 * 17 + 1)
                    assert np.array_equal(est[::2], oe) and np.array_equal(res[1::2], ores)
                    assert np.array_equal(conv[::2], oc) and np.array_equal(its[1::2], oi)
                    _, _, _, _, oq, orr = oracle.decode(g, cfg, syn1[17], segs)
                    assert np.array_equal(_bits(q), _bits(oq)) and np.array_equal(_bits(r), _bits(orr))
                assert_matches_oracle(oracle, g, cfg, syn1[:5], segs, dec=dec, messages=True)


@pytest.mark.parametrize("mode", REF_MODES)
@pytest.mark.parametrize("alpha", [1.0, 0.5])
def test_exact_zeros_ties_and_signed_zero_messages(oracle, mode, alpha):
    """Zeros and ties in the check update (proj/tests/test_decoder.cpp:207-221 tests the
    reference's two-minimum trick on them): with alpha a power of two and small integer
    priors of both signs the sums cancel exactly, so messages of +0.0 / -0.0 / 0 and tied
    minima occur at once.  Outcomes and every edge message (bit patterns: the sign of a zero
    included) must equal the oracle's - single-shot kernels, batch kernels, and the generic
    CSR kernel."""
    rng = np.random.default_rng(97)
    code = codes.make_code("bb72")
    cases = [(code.combined_graph, code.segments, 24),
             (codes.build_tanner_graph(codes.toy_code_3x6()), None, 8),
             (codes.build_tanner_graph(random_ldpc_matrix(rng, 9, 16)), None, 16)]
    zeros_seen = 0
    for g, segs, shots in cases:
        pri = rng.choice(np.array([-2.0, -1.0, 1.0, 1.0, 2.0, 3.0]), size=g.num_vars)
        syn = gf2.pack_bits((rng.random((shots, g.num_checks)) < 0.3).astype(np.uint8))
        for iters, early in ((9, True), (6, False)):
            cfg = DecoderConfig(max_iterations=iters, early_termination=early, alpha=alpha,
                                arithmetic=mode, priors=pri.tolist(),
                                quant_scale=0.0 if mode == "float" else 1.0)
            with Decoder(g, cfg, segments=segs) as dec:
                assert_matches_oracle(oracle, g, cfg, syn, segs, dec=dec, messages=True)
                dec.set_option(0, 1)  # the generic kernel, same handle
                assert_matches_oracle(oracle, g, cfg, syn[:4], segs, dec=dec, messages=True)
                dec.set_option(0, 0)
                oe, ores, oc, oi = oracle.decode_many(g, cfg, syn, segs)
                est, res, conv, its = dec.decode_batch_segments(syn)
                assert np.array_equal(est, oe) and np.array_equal(res, ores)
                assert np.array_equal(conv, oc) and np.array_equal(its, oi)
                if dec.get_option(INFO_BATCH_REGULAR) == 1:
                    # the regular batch kernels' own messages, general-prior instantiations
                    # (pairs of identical shots: both lanes of a packed pair stop together)
                    syn2 = np.repeat(syn, 2, axis=0)
                    for k in (0, 5):
                        q, r = dec.decode_batch_debug(syn2, 2 * k + 1)[4:]
                        _, _, _, _, oq, orr = oracle.decode(g, cfg, syn[k], segs)
                        assert np.array_equal(_bits(q), _bits(oq)) and np.array_equal(_bits(r), _bits(orr))
            for s in syn[:6]:
                _, _, _, _, oq, orr = oracle.decode(g, cfg, s, segs)
                zeros_seen += int((np.asarray(oq) == 0).sum() + (np.asarray(orr) == 0).sum())
    assert zeros_seen > 0, "the construction must produce zero messages"


@pytest.mark.parametrize("mode", REF_MODES)
@pytest.mark.parametrize("alpha", [0.5, 1.0, 0.25])
def test_uniform_prior_fast_paths_with_zero_messages(oracle, mode, alpha):
    """The uniform-prior instantiations (first iteration by table / from the syndrome) when
    the arithmetic produces exact zeros: gamma = 1 and alpha = 0.5 give q = 0.5 - 0.5 = +0.0
    already in the first iteration, whose magnitude then wins every minimum and whose sign
    travels through the products.  Batch kernels (messages of selected shots) and single-shot
    kernels against the oracle, bit patterns included."""
    code = codes.make_code("bb144")
    g = code.combined_graph
    rng = np.random.default_rng(int(alpha * 100))
    _, _, syn1 = error_syndromes(code, rng, 48, 0.04)
    syn = np.repeat(syn1, 2, axis=0)
    for iters, early in ((12, True), (5, False)):
        cfg = DecoderConfig(max_iterations=iters, early_termination=early, alpha=alpha, arithmetic=mode,
                            quant_scale=0.0 if mode == "float" else 2.0)
        oe, ores, oc, oi = oracle.decode_many(g, cfg, syn1, code.segments)
        with Decoder(code, cfg) as dec:
            for k in (0, 7, 30, 47):
                est, res, conv, its, q, r = dec.decode_batch_debug(syn, 2 * k)
                assert np.array_equal(est[::2], oe) and np.array_equal(res[1::2], ores)
                assert np.array_equal(conv[::2], oc) and np.array_equal(its[1::2], oi)
                _, _, _, _, oq, orr = oracle.decode(g, cfg, syn1[k], code.segments)
                assert np.array_equal(_bits(q), _bits(oq)), (k, "q")
                assert np.array_equal(_bits(r), _bits(orr)), (k, "r")
            assert_matches_oracle(oracle, g, cfg, syn1[:8], code.segments, dec=dec, messages=True)
    if alpha == 0.5:  # after the first iteration a variable with two unsatisfied checks sends 0
        one = DecoderConfig(max_iterations=1, early_termination=False, alpha=alpha, arithmetic=mode,
                            quant_scale=0.0 if mode == "float" else 2.0)
        zeros = 0
        with Decoder(code, one) as dec:
            for k in range(12):
                _, _, _, _, oq, _ = oracle.decode(g, one, syn1[k], code.segments)
                zeros += int((np.asarray(oq) == 0).sum())
                q = dec.decode_batch_debug(syn, 2 * k + 1)[4]
                assert np.array_equal(_bits(q), _bits(oq))
        assert zeros > 0, "alpha = 0.5 must produce zero messages in the first iteration"
