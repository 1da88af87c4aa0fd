"""BASELINE config 5 as named: phenomenological noise with SOFT (noisy) syndromes.

The reference takes priors per Decoder (proj/include/qldpc/decoder.hpp:31-32,
proj/src/decoder.cpp:108-131), so per-shot soft information means one Decoder per shot on
the extended graph [H | I] with priors = (LLR_data ..., |l_m| ...) and hard bits [l_m < 0]
(the identity columns take the degree-1-variable path, decoder.cpp:324-329).
qb_decode_batch_soft must reproduce exactly that: every outcome equal to the oracle's and to
the compiled reference's per-shot Decoder, for float, int8 and int16."""
import math

import numpy as np
import pytest

from paper_2508_07879_b200 import Decoder, DecoderConfig, codes, gf2
from paper_2508_07879_b200.campaign import PhenomenologicalCampaign

pytestmark = pytest.mark.gpu


def _ext(name):
    code = codes.make_code(name)
    h, segs = codes.extended_graph(code)
    return code, h, codes.build_tanner_graph(h), segs


def _soft_shots(code, h, g, rng, shots, p, mu, sigma):
    """numpy statement of the soft channel: data flips at p, l_m = (1 - 2 s~_m) mu + N(0, sigma^2)."""
    n, mz, mx = code.n, code.hz.rows, code.hx.rows
    data = np.zeros(g.num_vars, dtype=bool)
    data[:n] = True
    data[n + mz:2 * n + mz] = True
    err = ((rng.random((shots, g.num_vars)) < p) & data[None, :]).astype(np.uint8)
    s0 = h.mat_vec(err)
    l = (1.0 - 2.0 * s0) * mu + sigma * rng.standard_normal(s0.shape)
    s = (l < 0).astype(np.uint8)
    llr = 2.0 * mu * np.abs(l) / sigma ** 2
    flips = s ^ s0
    meas_vars = np.concatenate([np.arange(n, n + mz), np.arange(2 * n + mz, 2 * n + mz + mx)])
    err[:, meas_vars] = flips
    return err, s, llr


def _priors(code, p, mu, sigma):
    n, mz, mx = code.n, code.hz.rows, code.hx.rows
    llr_d = math.log((1 - p) / p)
    llr_m = 2 * mu * mu / sigma ** 2  # any value: replaced per shot
    return np.concatenate([np.full(n, llr_d), np.full(mz, llr_m), np.full(n, llr_d), np.full(mx, llr_m)])


def _dequant(dec, soft):
    cfg = dec.config()
    if cfg.arithmetic in ("float", "half"):
        return soft.astype(np.float64)
    scale = cfg.quant_scale or (8.0 if cfg.arithmetic == "int8" else 256.0)
    return soft.astype(np.float64) / scale


@pytest.mark.parametrize("mode,name,shots", [("float", "bb784", 2000), ("int8", "bb784", 2000),
                                             ("int16", "bb144", 600), ("int8", "bb144", 601)])
def test_soft_batch_equals_oracle_and_per_shot_reference(oracle, ref, mode, name, shots):
    code, h, g, segs = _ext(name)
    p, mu, sigma = 0.004, 1.0, 0.45
    rng = np.random.default_rng(11)
    err, s, llr = _soft_shots(code, h, g, rng, shots, p, mu, sigma)
    syn = gf2.pack_bits(s)
    cfg = DecoderConfig(max_iterations=30, arithmetic=mode, priors=_priors(code, p, mu, sigma).tolist())
    with Decoder(g, cfg, segments=segs) as dec:
        sv = dec.soft_vars()
        assert (sv != 0xffffffff).all() and len(set(sv.tolist())) == g.num_checks
        soft = dec.quantize_soft(llr)
        est, res, conv, its = dec.decode_batch_soft_segments(syn, soft)
        plain = dec.decode_batch_segments(syn[:64])  # the per-decoder priors still work afterwards
        again = dec.decode_batch_soft_segments(syn[:65], soft[:65])
        dq = _dequant(dec, soft)
    oe, ores, oc, oi = oracle.decode_many_soft(g, cfg, syn, sv, dq, segs)
    assert np.array_equal(est, oe) and np.array_equal(res, ores)
    assert np.array_equal(conv, oc) and np.array_equal(its, oi)
    assert np.array_equal(again[0], oe[:65]) and np.array_equal(again[3], oi[:65])
    pe, _, pc, pi = oracle.decode_many(g, cfg, syn[:64], segs)
    assert np.array_equal(plain[0], pe) and np.array_equal(plain[3], pi)
    # the unmodified reference, one Decoder per shot: its graph constructor makes ONE segment
    rg = ref.graph_from_coo(h.rows, h.cols, h.coo())
    m = min(shots, 500)
    rest, rres, rconv, rits = ref.decode_many_soft(rg, cfg, syn[:m], sv, dq[:m])
    with Decoder(g, cfg) as dec1:
        e1, r1, c1, i1 = dec1.decode_batch_soft_segments(syn[:m], soft[:m])
    assert np.array_equal(e1, rest) and np.array_equal(r1, rres)
    assert np.array_equal(c1[:, 0], rconv) and np.array_equal(i1[:, 0], rits)
    assert conv.min(axis=1).mean() > 0.5  # the point is in the decodable regime


def test_soft_information_matters_and_half_mode_runs():
    """The per-shot priors are really used: replacing them by their mean changes outcomes;
    half mode (no reference counterpart) decodes the same shots with a similar success rate."""
    code, h, g, segs = _ext("bb144")
    p, mu, sigma = 0.01, 1.0, 0.6
    rng = np.random.default_rng(5)
    err, s, llr = _soft_shots(code, h, g, rng, 4000, p, mu, sigma)
    syn = gf2.pack_bits(s)
    pri = _priors(code, p, mu, sigma)
    out = {}
    for mode in ("float", "half"):
        cfg = DecoderConfig(max_iterations=30, arithmetic=mode, priors=pri.tolist())
        with Decoder(g, cfg, segments=segs) as dec:
            soft = dec.quantize_soft(llr)
            out[mode] = dec.decode_batch_soft_segments(syn, soft)
            flat = dec.decode_batch_soft_segments(syn, np.full_like(soft, soft.mean()))
        if mode == "float":
            assert not np.array_equal(out[mode][0], flat[0])
            ok_soft = (gf2.unpack_bits(out[mode][0], g.num_vars) == err).all(axis=1).mean()
            ok_flat = (gf2.unpack_bits(flat[0], g.num_vars) == err).all(axis=1).mean()
            assert ok_soft > ok_flat  # soft information helps
    cf, ch = out["float"][2].min(axis=1).mean(), out["half"][2].min(axis=1).mean()
    assert abs(cf - ch) < 0.02


def test_soft_requires_the_degree_padded_kernel_and_valid_values():
    code = codes.make_code("bb72")
    with Decoder(code, DecoderConfig()) as dec:
        syn = np.zeros((4, gf2.num_words(dec.num_checks())), dtype=np.uint64)
        with pytest.raises(ValueError, match="degree-padded"):
            dec.decode_batch_soft_segments(syn, np.ones((4, dec.num_checks()), dtype=np.float32))
    _, h, g, segs = _ext("bb72")
    with Decoder(g, DecoderConfig(arithmetic="int8"), segments=segs) as dec:
        syn = np.zeros((4, gf2.num_words(g.num_checks)), dtype=np.uint64)
        with pytest.raises(ValueError, match="quantised prior is 0"):
            dec.decode_batch_soft_segments(syn, np.zeros((4, g.num_checks), dtype=np.int8))
        with pytest.raises(ValueError, match="soft values must be"):
            dec.decode_batch_soft_segments(syn, np.ones((4, 3), dtype=np.int8))
        est, _, conv, its = dec.decode_batch_soft_segments(syn, np.ones((4, g.num_checks), dtype=np.int8))
        assert not est.any() and conv.all() and (its == 1).all()
        assert dec.quantize_soft(np.array([0.0, 0.01, 0.06, 0.07, 100.0])).tolist() == [1, 1, 1, 1, 127]


def test_device_soft_generator_is_consistent_and_partition_independent():
    """qb_generate_soft_syndromes: H_ext * error == syndrome, flip rate of the channel
    = Phi(-mu / sigma), soft values are the quantised 2 mu |l| / sigma^2, and shot i only
    depends on (seed, first_trial + i)."""
    import torch
    code, h, g, segs = _ext("bb144")
    p, mu, sigma = 0.01, 1.0, 0.5
    shots = 20000
    sw, ew = gf2.num_words(g.num_checks), gf2.num_words(g.num_vars)
    n, mz = code.n, code.hz.rows
    for mode, dt in (("float", torch.float32), ("int8", torch.int8)):
        cfg = DecoderConfig(max_iterations=20, arithmetic=mode, priors=_priors(code, p, mu, sigma).tolist())
        d_syn = torch.zeros((shots, sw), dtype=torch.int64, device="cuda")
        d_err = torch.zeros((shots, ew), dtype=torch.int64, device="cuda")
        d_soft = torch.zeros((shots, g.num_checks), dtype=dt, device="cuda")
        st = torch.cuda.current_stream().cuda_stream
        with Decoder(g, cfg, segments=segs) as dec:
            dec.generate_soft_syndromes(3, p, mu, sigma, shots, d_syn.data_ptr(), d_soft.data_ptr(),
                                        d_err.data_ptr(), stream=st)
            torch.cuda.synchronize()
            syn = gf2.unpack_bits(d_syn.cpu().numpy().view(np.uint64), g.num_checks)
            err = gf2.unpack_bits(d_err.cpu().numpy().view(np.uint64), g.num_vars)
            soft = d_soft.cpu().numpy()
            # a second call shifted by 777 trials reproduces the tail of the first
            d_syn2 = torch.zeros((100, sw), dtype=torch.int64, device="cuda")
            d_soft2 = torch.zeros((100, g.num_checks), dtype=dt, device="cuda")
            dec.generate_soft_syndromes(3, p, mu, sigma, 100, d_syn2.data_ptr(), d_soft2.data_ptr(),
                                        None, first_trial=777, stream=st)
            torch.cuda.synchronize()
            assert torch.equal(d_syn2, d_syn[777:877]) and torch.equal(d_soft2, d_soft[777:877])
            est, res, conv, its = dec.decode_batch_soft_segments(
                d_syn[:3000].cpu().numpy().view(np.uint64), soft[:3000])
        assert np.array_equal(syn, h.mat_vec(err))
        meas = np.concatenate([err[:, n:n + mz], err[:, 2 * n + mz:]], axis=1)
        q = 0.5 * math.erfc(mu / sigma / math.sqrt(2))
        assert abs(meas.mean() - q) < 5 * math.sqrt(q * (1 - q) / meas.size)
        data = np.concatenate([err[:, :n], err[:, n + mz:2 * n + mz]], axis=1)
        assert abs(data.mean() - p) < 5 * math.sqrt(p * (1 - p) / data.size)
        if mode == "float":
            # E|l| of a folded normal with mean mu, sd sigma
            ea = sigma * math.sqrt(2 / math.pi) * math.exp(-mu * mu / (2 * sigma * sigma)) + \
                mu * (1 - 2 * q)
            assert abs(soft.mean() / (2 * mu / sigma ** 2) - ea) < 0.01
            assert (soft >= 0).all()
        else:
            assert soft.min() >= 1 and soft.max() <= 127
        assert conv.min(axis=1).mean() > 0.9


@pytest.mark.parametrize("mode", ["int8", "float"])
def test_device_campaigns_on_the_extended_graph(mode):
    """qb_campaign_run (hard noisy syndromes) and qb_campaign_run_soft on the extended graph:
    the ten counters equal the host's classification of the same generate + decode, and do
    not depend on how the trials are split over calls."""
    import torch
    code = codes.make_code("bb144")
    p, q, mu, sigma = 0.015, 0.015, 1.0, 0.5
    trials = 6000
    camp = PhenomenologicalCampaign(code, DecoderConfig(max_iterations=30, arithmetic=mode), p, q)
    try:
        dec, g = camp.decoder, camp.graph
        sw, ew = gf2.num_words(g.num_checks), gf2.num_words(g.num_vars)
        d_syn = torch.zeros((trials, sw), dtype=torch.int64, device="cuda")
        d_err = torch.zeros((trials, ew), dtype=torch.int64, device="cuda")
        st = torch.cuda.current_stream().cuda_stream
        # ---- hard
        whole = camp.run_range(9, 0, trials)
        parts = camp.run_range(9, 0, 2500) + camp.run_range(9, 2500, trials - 2500)
        assert np.array_equal(whole, parts)
        dec.generate_syndromes(9, 0.0, trials, d_syn.data_ptr(), d_err.data_ptr(), probs=camp.probs,
                               css_interleave=False, stream=st)
        torch.cuda.synchronize()
        syn_w = d_syn.cpu().numpy().view(np.uint64)
        est, _, conv, its = dec.decode_batch_segments(syn_w, want_residual=False)
        host = camp.host_counters(gf2.unpack_bits(d_err.cpu().numpy().view(np.uint64), g.num_vars),
                                  gf2.unpack_bits(est, g.num_vars), conv, its,
                                  gf2.unpack_bits(syn_w, g.num_checks))
        assert np.array_equal(whole, host), (whole, host)
        assert whole[9] == trials and whole[2] + whole[3] + whole[4] + whole[5] > 0
        # ---- soft
        swhole = camp.run_range_soft(9, mu, sigma, 0, trials)
        sparts = camp.run_range_soft(9, mu, sigma, 0, 1000) + camp.run_range_soft(9, mu, sigma, 1000, trials - 1000)
        assert np.array_equal(swhole, sparts)
        d_soft = torch.zeros((trials, g.num_checks), device="cuda",
                             dtype=torch.int8 if mode == "int8" else torch.float32)
        dec.generate_soft_syndromes(9, p, mu, sigma, trials, d_syn.data_ptr(), d_soft.data_ptr(),
                                    d_err.data_ptr(), stream=st)
        torch.cuda.synchronize()
        syn_w = d_syn.cpu().numpy().view(np.uint64)
        est, _, conv, its = dec.decode_batch_soft_segments(syn_w, d_soft.cpu().numpy(), want_residual=False)
        host = camp.host_counters(gf2.unpack_bits(d_err.cpu().numpy().view(np.uint64), g.num_vars),
                                  gf2.unpack_bits(est, g.num_vars), conv, its,
                                  gf2.unpack_bits(syn_w, g.num_checks))
        assert np.array_equal(swhole, host), (swhole, host)
    finally:
        camp.close()


@pytest.mark.parametrize("mode", ["float", "int8", "int16"])
def test_single_shot_soft_decode_in_every_io_protocol(oracle, mode):
    """qb_decode_soft: per-shot priors through the single-shot cluster kernel
    (decode_ell_latency_kernel) with the syndrome in the kernel parameters, by memcpy and by
    doorbell, interleaved with plain single shots on the same handle; outcomes equal the
    oracle's per-shot-prior decode and the batch call's."""
    code, h, g, segs = _ext("bb144")
    p, mu, sigma = 0.006, 1.0, 0.45
    rng = np.random.default_rng(19)
    err, s, llr = _soft_shots(code, h, g, rng, 40, p, mu, sigma)
    syn = gf2.pack_bits(s)
    cfg = DecoderConfig(max_iterations=25, arithmetic=mode, priors=_priors(code, p, mu, sigma).tolist())
    with Decoder(g, cfg, segments=segs) as dec:
        sv = dec.soft_vars()
        soft = dec.quantize_soft(llr)
        want = oracle.decode_many_soft(g, cfg, syn, sv, _dequant(dec, soft), segs)
        plain = oracle.decode_many(g, cfg, syn, segs)
        batch = dec.decode_batch_soft_segments(syn, soft)
        assert all(np.array_equal(a, b) for a, b in zip(batch, want))
        for io_mode in (0, 1, 2):
            dec.set_option(1, io_mode)
            launches = dec.launch_count()
            for k in range(len(syn)):
                one = dec.decode_soft_segments(syn[k], soft[k])
                assert all(np.array_equal(a, b[k]) for a, b in zip(one, want)), (io_mode, k)
            if io_mode == 2:
                assert dec.launch_count() - launches <= 2, "doorbell mode must not launch per shot"
            for k in (0, 5):  # plain single shots in between (the decoder's own priors)
                one = dec.decode_segments(syn[k])
                assert all(np.array_equal(a, b[k]) for a, b in zip(one, plain)), (io_mode, k, "plain")
            one = dec.decode_soft_segments(syn[7], soft[7])
            assert all(np.array_equal(a, b[7]) for a, b in zip(one, want))
    with Decoder(codes.make_code("bb72"), DecoderConfig()) as dec:
        with pytest.raises(ValueError, match="degree-padded"):
            dec.decode_soft_segments(np.zeros(gf2.num_words(dec.num_checks()), dtype=np.uint64),
                                     np.ones(dec.num_checks(), dtype=np.float32))


@pytest.mark.parametrize("mode", ["float", "int8", "int16"])
def test_soft_decode_matches_the_golden_fixture_of_the_compiled_reference(mode):
    """tests/golden/soft_bb144_p0.01.npz holds the outcomes of one UNMODIFIED reference Decoder
    per shot (generated in the authoring container, tests/golden/make_golden.py): the batch
    kernel and the single-shot kernel, handed the stored reliabilities, reproduce them."""
    import os
    d = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "soft_bb144_p0.01.npz"))
    code = codes.make_code(str(d["code"]))
    h, segs = codes.extended_graph(code)
    g = codes.build_tanner_graph(h)
    cfg = DecoderConfig(max_iterations=int(d["max_iterations"]), arithmetic=mode,
                        priors=[float(d["prior_data"])] * g.num_vars)
    syn, soft = d["syndromes"], d[f"{mode}_soft"]
    with Decoder(g, cfg, segments=segs) as dec:
        assert np.array_equal(dec.soft_vars(), d["soft_vars"])
        assert np.array_equal(dec.quantize_soft(d["llr"]), soft)
        est, res, conv, its = dec.decode_batch_soft_segments(syn, soft)
        assert np.array_equal(est, d[f"{mode}_estimate"]) and np.array_equal(res, d[f"{mode}_residual"])
        assert np.array_equal(conv.min(axis=1), d[f"{mode}_converged"])
        assert np.array_equal(its.max(axis=1), d[f"{mode}_iterations"])
        for io_mode in (0, 2):
            dec.set_option(1, io_mode)
            for k in range(0, len(syn), 5):
                e1, r1, c1, i1 = dec.decode_soft_segments(syn[k], soft[k])
                assert np.array_equal(e1, d[f"{mode}_estimate"][k]) and np.array_equal(r1, d[f"{mode}_residual"][k])
                assert c1.min() == d[f"{mode}_converged"][k] and i1.max() == d[f"{mode}_iterations"][k]
