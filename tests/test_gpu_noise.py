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
