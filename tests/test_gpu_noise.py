"""Device noise/syndrome generator and bench-protocol parity against the
compiled reference (prebuilt oracle/_ref): the generator must reproduce
`sample_error` + `extract_syndromes` bit for bit, and the latency harness must
reproduce `run_bench`'s FNV-1a output digest."""
import numpy as np
import pytest

from paper_2508_07879_b200 import Decoder, DecoderConfig, codes, gf2

pytestmark = pytest.mark.gpu


def _generate(dec, code, seed, p, shots, first_trial=0):
    import torch
    g = code.combined_graph
    sw, ew = gf2.num_words(g.num_checks), gf2.num_words(g.num_vars)
    d_syn = torch.zeros((shots, sw), dtype=torch.int64, device="cuda")
    d_err = torch.zeros((shots, ew), dtype=torch.int64, device="cuda")
    dec.generate_syndromes(seed, p, shots, d_syn.data_ptr(), d_err.data_ptr(),
                           first_trial=first_trial, stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return d_syn.cpu().numpy().view(np.uint64), d_err.cpu().numpy().view(np.uint64)


@pytest.mark.parametrize("name", ["bb72", "bb784"])
def test_generator_reproduces_reference_sampler(ref, name):
    """proj/src/noise.cpp:23-26, :67-78 (SplitMix64 per-trial streams) and :97-105."""
    code = codes.make_code(name)
    rc = ref.code(name)
    with Decoder(code, DecoderConfig()) as dec:
        for seed, p, first in ((1, 0.01, 0), (12345, 0.05, 1000), (0xACCE5501, 0.3, 7)):
            syn, err = _generate(dec, code, seed, p, 200, first)
            rsyn, rex, rez = ref.syndrome_pool(rc, p, seed, 200, first_trial=first, with_errors=True)
            assert np.array_equal(syn, rsyn)
            ebits = gf2.unpack_bits(err, 2 * code.n)
            assert np.array_equal(ebits[:, :code.n], gf2.unpack_bits(rex, code.n))
            assert np.array_equal(ebits[:, code.n:], gf2.unpack_bits(rez, code.n))


def test_generator_marginals_and_syndrome_map():
    """Statistical + structural checks that need no reference: flip rate within
    4 sigma, syndrome == H * error for every shot (proj/tests/test_noise.cpp:125-219)."""
    code = codes.make_code("bb144")
    g = code.combined_graph
    with Decoder(code, DecoderConfig()) as dec:
        syn, err = _generate(dec, code, 99, 0.05, 20000)
    ebits = gf2.unpack_bits(err, g.num_vars)
    n = ebits.size
    assert abs(ebits.mean() - 0.05) < 4 * np.sqrt(0.05 * 0.95 / n)
    assert np.array_equal(gf2.unpack_bits(syn, g.num_checks), code.combined.mat_vec(ebits))


def _generate_opt(dec, g, seed, p, shots, first_trial=0, probs=None, css=True):
    import torch
    sw, ew = gf2.num_words(g.num_checks), gf2.num_words(g.num_vars)
    d_syn = torch.full((shots, sw), -1, dtype=torch.int64, device="cuda")
    d_err = torch.full((shots, ew), -1, dtype=torch.int64, device="cuda")
    dec.generate_syndromes(seed, p, shots, d_syn.data_ptr(), d_err.data_ptr(), first_trial=first_trial,
                           probs=probs, css_interleave=css,
                           stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return d_syn.cpu().numpy().view(np.uint64), d_err.cpu().numpy().view(np.uint64)


@pytest.mark.parametrize("name,p,shots", [("bb144", 0.05, 20000), ("bb784", 0.01, 30001),
                                          ("bb72", 0.3, 5000)])
def test_skip_sampler_has_the_bernoulli_distribution(name, p, shots):
    """QB_OPT_SAMPLER = 1 (geometric gaps, one draw per flip) is a different stream with the
    same law as sample_error's independent-xz model (proj/src/noise.cpp:73-77): syndrome ==
    H * error on every shot, padding bits clear, per-variable and overall flip rates, the
    weight's mean AND variance (a gap-law error would show there), neighbour correlation."""
    from paper_2508_07879_b200 import _lib
    code = codes.make_code(name)
    g = code.combined_graph
    n = g.num_vars
    with Decoder(code, DecoderConfig()) as dec:
        dec.set_option(_lib.OPT_SAMPLER, 1)
        assert dec.get_option(_lib.OPT_SAMPLER) == 1
        syn, err = _generate_opt(dec, g, 7, p, shots)
        again, _ = _generate_opt(dec, g, 7, p, shots)
        head, _ = _generate_opt(dec, g, 7, p, 100, first_trial=shots - 100)
        other, _ = _generate_opt(dec, g, 8, p, shots)
        dec.set_option(_lib.OPT_SAMPLER, 0)
        exact, _ = _generate_opt(dec, g, 7, p, 64)
    assert np.array_equal(syn, again)                      # deterministic in (seed, trial)
    assert np.array_equal(head, syn[shots - 100:])         # keyed by trial, not by launch shape
    assert not np.array_equal(other, syn) and not np.array_equal(exact, syn[:64])
    ebits = gf2.unpack_bits(err, n)
    assert np.array_equal(gf2.pack_bits(ebits), err)       # no bit set beyond N
    assert np.array_equal(gf2.unpack_bits(syn, g.num_checks), code.combined.mat_vec(ebits))
    assert np.array_equal(gf2.pack_bits(gf2.unpack_bits(syn, g.num_checks)), syn)
    sd1 = np.sqrt(p * (1 - p))
    assert abs(ebits.mean() - p) < 4 * sd1 / np.sqrt(ebits.size)
    per_var = ebits.mean(axis=0)
    assert np.abs(per_var - p).max() < 5 * sd1 / np.sqrt(shots)   # incl. the first and last variable
    w = ebits.sum(axis=1).astype(np.float64)
    assert abs(w.mean() - n * p) < 4 * np.sqrt(n * p * (1 - p) / shots)
    var = n * p * (1 - p)
    # Var of the sample variance of a binomial ~ 2 var^2 / shots (+ small kurtosis term)
    assert abs(w.var() - var) < 5 * var * np.sqrt(2.0 / shots) + 0.01 * var
    c = ((ebits[:, 1:] - p) * (ebits[:, :-1] - p)).mean() / (p * (1 - p))
    assert abs(c) < 4 / np.sqrt(ebits[:, 1:].size)


def test_skip_sampler_equals_its_plain_python_statement():
    """The kernel against tests/helpers.skip_sampler_flips (same counter-based stream, same
    gap formula in fp64) on the first trials of two ranges."""
    from paper_2508_07879_b200 import _lib
    from tests.helpers import skip_sampler_flips
    code = codes.make_code("bb144")
    g = code.combined_graph
    with Decoder(code, DecoderConfig()) as dec:
        dec.set_option(_lib.OPT_SAMPLER, 1)
        for seed, p, first in ((1, 0.01, 0), (12345, 0.2, 1000)):
            _, err = _generate_opt(dec, g, seed, p, 150, first_trial=first)
            ebits = gf2.unpack_bits(err, g.num_vars)
            for i in range(150):
                assert np.flatnonzero(ebits[i]).tolist() == skip_sampler_flips(
                    seed, first + i, p, g.num_vars), (seed, i)


def test_skip_sampler_edge_probabilities_and_thinning():
    """p = 0 flips nothing, p = 1 flips everything; per-variable probabilities (thinning at
    p_max) reproduce each class's rate on the extended [H | I] graph of BASELINE config 5."""
    from paper_2508_07879_b200 import _lib
    from tests.test_gpu_phenomenological import _setup
    code = codes.make_code("bb72")
    g = code.combined_graph
    with Decoder(code, DecoderConfig()) as dec:
        dec.set_option(_lib.OPT_SAMPLER, 1)
        syn0, err0 = _generate_opt(dec, g, 3, 0.0, 257)
        syn1, err1 = _generate_opt(dec, g, 3, 1.0, 257)
    assert not syn0.any() and not err0.any()
    assert gf2.unpack_bits(err1, g.num_vars).all()
    ones = np.ones((1, g.num_vars), dtype=np.uint8)
    assert np.array_equal(gf2.unpack_bits(syn1, g.num_checks),
                          np.repeat(code.combined.mat_vec(ones), 257, axis=0))
    code, h, g, segs, priors, probs = _setup("bb144", 0.03, 0.01)
    shots = 20000
    cfg = DecoderConfig(max_iterations=20, arithmetic="int8", priors=priors.tolist())
    with Decoder(g, cfg, segments=segs) as dec:
        dec.set_option(_lib.OPT_SAMPLER, 1)
        syn, err = _generate_opt(dec, g, 5, 0.0, shots, probs=probs, css=False)
    e = gf2.unpack_bits(err, g.num_vars)
    assert np.array_equal(gf2.unpack_bits(syn, g.num_checks), h.mat_vec(e))
    for lo, hi, pr in ((0, code.n, 0.03), (code.n, code.n + code.hz.rows, 0.01)):
        part = e[:, lo:hi]
        assert abs(part.mean() - pr) < 4 * np.sqrt(pr * (1 - pr) / part.size)
        assert np.abs(part.mean(axis=0) - pr).max() < 5 * np.sqrt(pr * (1 - pr) / shots)


@pytest.mark.parametrize("mode", ["float", "int8"])
def test_latency_harness_digest_equals_reference_run_bench(ref, mode):
    """run_bench at batch 1 (proj/src/bench.cpp:182-337): same pool recipe, same
    decode order, same FNV-1a digest over (converged, iterations, estimate)."""
    name = "bb144"
    code = codes.make_code(name)
    rc = ref.code(name)
    for iters, early in ((10, False), (50, True)):
        r = ref.run_bench(rc, arithmetic=mode, max_iterations=iters, early_termination=early,
                          batch=1, threads=1, warmup=100, measure=200, p=0.02, seed=1)
        pool = ref.syndrome_pool(rc, 0.02, 1, 256)
        cfg = DecoderConfig(max_iterations=iters, early_termination=early, arithmetic=mode)
        with Decoder(code, cfg) as dec:
            for io_mode in (0, 1, 2):
                dec.set_option(1, io_mode)
                wall, kern, digest = dec.latency_run(pool, 100, 200)
                assert digest == r["digest"]
                assert (wall > 0).all() and (kern > 0).all()
