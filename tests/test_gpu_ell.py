"""GPU parity of the degree-padded (ELL) batch kernel (csrc/kernel_ell.cuh) — the
loader's path for IRREGULAR graphs: every check padded to DC slots with a
sentinel, every variable to DV slots pointing at a zero block.  Batches decoded
by it must equal the CPU oracle bit for bit in float / int8 / int16, equal the
generic CSR kernel in every mode (incl. half), and the compiled reference on the
same inputs.  Cases follow the reference's irregular-graph tests
(proj/tests/test_decoder.cpp:436-447: degree-1 checks and variables) plus the
degree patterns the padding must survive: degree-0 nodes, saturating priors,
segments that share packed words, more shots than resident CTAs."""
import numpy as np
import pytest

from paper_2508_07879_b200 import Decoder, DecoderConfig, codes, gf2
from tests.helpers import random_ldpc_matrix, random_syndromes

pytestmark = pytest.mark.gpu

REF_MODES = ("float", "int8", "int16")
OPT_KERNEL, OPT_INFO_ELL = 0, 107


def _batch(dec, syn):
    return dec.decode_batch_segments(syn)


def _same(a, b):
    return all(np.array_equal(x, y) for x, y in zip(a, b))


@pytest.mark.parametrize("mode", REF_MODES)
def test_random_irregular_graphs_equal_oracle(oracle, mode):
    """Random sparse graphs with degree-1 checks / variables, random priors."""
    rng = np.random.default_rng(2508)
    used = set()
    for trial in range(12):
        rows, cols = 8 + int(rng.integers(0, 40)), 12 + int(rng.integers(0, 60))
        h = random_ldpc_matrix(rng, rows, cols)
        g = codes.build_tanner_graph(h)
        priors = (rng.uniform(0.5, 6.0, g.num_vars) * rng.choice([-1.0, 1.0], g.num_vars, p=[0.1, 0.9]))
        cfg = DecoderConfig(alpha=0.8 if trial % 3 else 0.625, max_iterations=12,
                            early_termination=trial % 2 == 0, arithmetic=mode,
                            priors=priors.tolist() if trial % 4 else None)
        syn = random_syndromes(rng, 200, g.num_checks, 0.25)
        with Decoder(g, cfg) as dec:
            ell = dec.get_option(OPT_INFO_ELL)
            got = _batch(dec, syn)
        if ell:
            used.add(ell)
        want = oracle.decode_many(g, cfg, syn, None)
        assert _same(got, want), f"trial {trial}: ELL {ell} differs from the oracle"
    assert used, "no graph was served by the degree-padded kernel"


@pytest.mark.parametrize("mode", REF_MODES + ("half",))
def test_ell_equals_generic_kernel(mode):
    """Same handle, batch through the ELL kernel and through the generic CSR kernel."""
    rng = np.random.default_rng(11)
    for trial in range(6):
        h = random_ldpc_matrix(rng, 30 + int(rng.integers(0, 30)), 50 + int(rng.integers(0, 50)))
        g = codes.build_tanner_graph(h)
        priors = rng.uniform(0.3, 5.0, g.num_vars)
        cfg = DecoderConfig(max_iterations=15, early_termination=trial % 2 == 0, arithmetic=mode,
                            priors=priors.tolist())
        syn = random_syndromes(rng, 500, g.num_checks, 0.2)
        with Decoder(g, cfg) as dec:
            assert dec.get_option(OPT_INFO_ELL) != 0
            a = _batch(dec, syn)
            dec.set_option(OPT_KERNEL, 1)
            assert dec.get_option(OPT_INFO_ELL) == 0
            b = _batch(dec, syn)
        assert _same(a, b)


def _degree_zero_graph():
    # 5 checks x 9 variables: variable 4 has no check, check 3 has no variable,
    # check 0 has degree 1, variable 8 has degree 1
    dense = np.zeros((5, 9), dtype=np.uint8)
    dense[0, 0] = 1
    dense[1, [0, 1, 2, 3]] = 1
    dense[2, [1, 2, 5, 6, 7]] = 1
    dense[4, [3, 5, 6, 7, 8]] = 1
    return codes.SparseMatrix.from_dense(dense)


@pytest.mark.parametrize("mode", REF_MODES)
def test_degree_zero_and_degree_one_nodes(oracle, mode):
    h = _degree_zero_graph()
    g = codes.build_tanner_graph(h)
    syn = gf2.pack_bits(np.array([[(mask >> m) & 1 for m in range(5)] for mask in range(32)],
                                 dtype=np.uint8))
    for early in (True, False):
        cfg = DecoderConfig(max_iterations=9, early_termination=early, arithmetic=mode,
                            priors=[1.5, -0.75, 2.0, 0.5, -3.0, 1.0, 1.0, 4.0, 0.25])
        with Decoder(g, cfg) as dec:
            assert dec.get_option(OPT_INFO_ELL) != 0
            got = _batch(dec, syn)
        assert _same(got, oracle.decode_many(g, cfg, syn, None))


@pytest.mark.parametrize("mode", REF_MODES)
def test_toy_code_batches(oracle, mode):
    """toy 3x6 (check degree 4, variable degree 2): all 8 syndromes, many times over."""
    g = codes.build_tanner_graph(codes.toy_code_3x6())
    syn = gf2.pack_bits(np.array([[(mask >> m) & 1 for m in range(3)] for mask in range(8)] * 300,
                                 dtype=np.uint8))
    cfg = DecoderConfig(max_iterations=10, arithmetic=mode)
    with Decoder(g, cfg) as dec:
        assert dec.get_option(OPT_INFO_ELL) == 402
        got = _batch(dec, syn)
    assert _same(got, oracle.decode_many(g, cfg, syn, None))


@pytest.mark.parametrize("mode,scale", [("int8", 8.0), ("float", 0.0), ("int16", 256.0)])
def test_extended_bb784_two_segments(oracle, ref, mode, scale):
    """BASELINE config 5 at full size: diag([Hz | I], [Hx | I]) of [[784,24,24]], data
    flips p, measurement flips q, LLR priors; 2 segments whose packed words overlap."""
    code = codes.make_code("bb784")
    h, segs = codes.extended_graph(code)
    g = codes.build_tanner_graph(h)
    n, mz, mx = code.n, code.hz.rows, code.hx.rows
    p, q = 0.01, 0.02
    priors = np.concatenate([np.full(n, np.log((1 - p) / p)), np.full(mz, np.log((1 - q) / q)),
                             np.full(n, np.log((1 - p) / p)), np.full(mx, np.log((1 - q) / q))])
    probs = np.concatenate([np.full(n, p), np.full(mz, q), np.full(n, p), np.full(mx, q)])
    rng = np.random.default_rng(784)
    e = (rng.random((3000, g.num_vars)) < probs).astype(np.uint8)
    syn = gf2.pack_bits(h.mat_vec(e))
    cfg = DecoderConfig(max_iterations=30, arithmetic=mode, priors=priors.tolist(), quant_scale=scale)
    with Decoder(g, cfg, segments=segs) as dec:
        assert dec.get_option(OPT_INFO_ELL) == 703
        got = _batch(dec, syn)
        one = dec.decode_segments(syn[7])
    want = oracle.decode_many(g, cfg, syn[:400], segs)
    assert _same([x[:400] for x in got], want)
    assert np.array_equal(one[0], got[0][7]) and np.array_equal(one[3], got[3][7])
    # the whole batch against the generic kernel (oracle-checked above on a prefix)
    with Decoder(g, cfg, segments=segs) as dec:
        dec.set_option(OPT_KERNEL, 1)
        assert _same(got, _batch(dec, syn))
    # and the compiled reference (its graph constructor makes ONE segment)
    rg = ref.graph_from_coo(h.rows, h.cols, h.coo())
    rest, rres, rconv, rits = ref.decoder(rg, cfg).decode_many(syn[:300])
    with Decoder(g, cfg) as dec1:  # 784 checks x 2352 variables in one segment
        est1, res1, conv1, its1 = _batch(dec1, syn[:300])
    assert np.array_equal(est1, rest) and np.array_equal(res1, rres)
    assert np.array_equal(conv1[:, 0], rconv) and np.array_equal(its1[:, 0], rits)


def test_soundness_at_scale():
    """Size-independent property on 2^17 shots of the extended [[784,24,24]] graph:
    residual == H * e_hat xor s, and converged <=> residual == 0 per segment."""
    import torch
    code = codes.make_code("bb784")
    h, segs = codes.extended_graph(code)
    g = codes.build_tanner_graph(h)
    n, mz, mx = code.n, code.hz.rows, code.hx.rows
    p = q = 0.005
    llr = float(np.log((1 - p) / p))
    probs = np.full(g.num_vars, p)
    cfg = DecoderConfig(max_iterations=20, arithmetic="int8", priors=[llr] * g.num_vars)
    shots = 1 << 17
    sw, ew = gf2.num_words(g.num_checks), gf2.num_words(g.num_vars)
    d_syn = torch.zeros((shots, sw), dtype=torch.int64, device="cuda")
    d_est = torch.zeros((shots, ew), dtype=torch.int64, device="cuda")
    d_res = torch.zeros((shots, sw), dtype=torch.int64, device="cuda")
    d_conv = torch.zeros((shots, 2), dtype=torch.uint8, device="cuda")
    d_its = torch.zeros((shots, 2), dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    with Decoder(g, cfg, segments=segs) as dec:
        assert dec.get_option(OPT_INFO_ELL) == 703
        dec.generate_syndromes(3, 0.0, shots, d_syn.data_ptr(), None, probs=probs,
                               css_interleave=False, stream=stream)
        dec.decode_batch_device(shots, d_syn.data_ptr(), d_est.data_ptr(), d_res.data_ptr(),
                                d_conv.data_ptr(), d_its.data_ptr(), stream)
        torch.cuda.synchronize()
    sub = slice(0, 4096)
    syn = gf2.unpack_bits(d_syn[sub].cpu().numpy().view(np.uint64), g.num_checks)
    est = gf2.unpack_bits(d_est[sub].cpu().numpy().view(np.uint64), g.num_vars)
    res = gf2.unpack_bits(d_res[sub].cpu().numpy().view(np.uint64), g.num_checks)
    assert np.array_equal(res, h.mat_vec(est) ^ syn)
    res_all = d_res.cpu().numpy().view(np.uint64)
    bits_all = gf2.unpack_bits(res_all, g.num_checks)
    conv = d_conv.cpu().numpy()
    assert np.array_equal(conv[:, 0] == 1, ~bits_all[:, :mz].any(axis=1))
    assert np.array_equal(conv[:, 1] == 1, ~bits_all[:, mz:].any(axis=1))
    assert conv.mean() > 0.5


@pytest.mark.parametrize("mode", ["int8", "half"])
def test_packed_pairs_on_irregular_graphs(oracle, mode):
    """decode_ell_h2_kernel (two shots per thread on packed fp16 instructions): equal to the
    one-shot-per-thread degree-padded kernel and to the generic CSR kernel on the same
    handle; in int8 mode also to the integer oracle (decoder.cpp:260-283).  Odd shot counts
    exercise the half-empty last pair; the graphs have degree-0 / degree-1 nodes."""
    OPT_HALF_PAIRS = 10
    rng = np.random.default_rng(77)
    graphs = [codes.build_tanner_graph(_degree_zero_graph())]
    for _ in range(5):
        graphs.append(codes.build_tanner_graph(
            random_ldpc_matrix(rng, 20 + int(rng.integers(0, 60)), 40 + int(rng.integers(0, 80)))))
    paired = 0
    for gi, g in enumerate(graphs):
        priors = rng.uniform(0.2, 12.0, g.num_vars) * rng.choice([-1.0, 1.0], g.num_vars, p=[0.1, 0.9])
        for early in (True, False):
            cfg = DecoderConfig(max_iterations=11, early_termination=early, arithmetic=mode,
                                priors=priors.tolist(), alpha=0.8 if gi % 2 else 0.625)
            syn = random_syndromes(rng, 333, g.num_checks, 0.2)
            with Decoder(g, cfg) as dec:
                if not dec.get_option(OPT_INFO_ELL):
                    continue
                paired += dec.get_option(OPT_HALF_PAIRS)
                a = _batch(dec, syn)
                dec.set_option(OPT_HALF_PAIRS, 0)
                assert dec.get_option(OPT_HALF_PAIRS) == 0 and dec.get_option(OPT_INFO_ELL)
                assert _same(a, _batch(dec, syn)), "pairs vs one shot per thread"
                dec.set_option(OPT_KERNEL, 1)
                assert _same(a, _batch(dec, syn)), "pairs vs generic"
            if mode == "int8":
                assert _same(a, oracle.decode_many(g, cfg, syn, None)), "pairs vs oracle"
    assert paired >= 6, "the packed kernel was not selected"


@pytest.mark.parametrize("mode", REF_MODES)
def test_single_shots_through_the_degree_padded_kernel(oracle, mode):
    """qb_decode on irregular graphs runs decode_ell_latency_kernel - the degree-padded node
    updates inside the single-shot cluster protocol (one CTA per segment, one check per
    thread): every outcome, per segment, equals the oracle's in all three I/O settings
    (syndrome in the kernel parameters + mapped records, memcpy protocol, persistent
    doorbell without a launch per shot), interleaved with batches on the same handle; the
    final edge messages (qb_decode_debug) match bit for bit."""
    OPT_LATENCY_IO = 1
    code = codes.make_code("bb144")
    h, segs = codes.extended_graph(code)
    g = codes.build_tanner_graph(h)
    rng = np.random.default_rng(31)
    probs = np.full(g.num_vars, 0.02)
    e = (rng.random((60, g.num_vars)) < probs).astype(np.uint8)
    syn = gf2.pack_bits(h.mat_vec(e))
    priors = rng.uniform(1.0, 6.0, g.num_vars)
    for early in (True, False):
        cfg = DecoderConfig(max_iterations=12, early_termination=early, arithmetic=mode,
                            priors=priors.tolist())
        want = oracle.decode_many(g, cfg, syn, segs)
        with Decoder(g, cfg, segments=segs) as dec:
            assert dec.get_option(106) == 1 and dec.get_option(103) == 1  # cluster kernel in use
            for io_mode in (0, 1, 2):
                dec.set_option(OPT_LATENCY_IO, io_mode)
                launches = dec.launch_count()
                for k in range(len(syn)):
                    one = dec.decode_segments(syn[k])
                    assert all(np.array_equal(a, b[k]) for a, b in zip(one, want)), (io_mode, k)
                    assert dec.last_kernel_ns() > 0
                if io_mode == 2:
                    assert dec.launch_count() - launches <= 2, "doorbell mode must not launch per shot"
                assert _same(_batch(dec, syn), want)
            dec.set_option(OPT_LATENCY_IO, 0)
            for k in (0, 17, 59):
                est, res, conv, its, q, r = dec.decode_debug(syn[k])
                _, _, _, oi, oq, orr = oracle.decode(g, cfg, syn[k], segs)
                assert np.array_equal(its, oi)
                assert np.array_equal(q.view(np.uint32), oq.view(np.uint32))
                assert np.array_equal(r.view(np.uint32), orr.view(np.uint32))
    # irregular single-segment graphs with degree-0 / degree-1 nodes
    for g2 in (codes.build_tanner_graph(_degree_zero_graph()),
               codes.build_tanner_graph(random_ldpc_matrix(rng, 25, 60))):
        cfg = DecoderConfig(max_iterations=9, arithmetic=mode,
                            priors=rng.uniform(0.3, 4.0, g2.num_vars).tolist())
        syn2 = random_syndromes(rng, 40, g2.num_checks, 0.3)
        want = oracle.decode_many(g2, cfg, syn2, None)
        with Decoder(g2, cfg) as dec:
            for io_mode in (0, 2):
                dec.set_option(OPT_LATENCY_IO, io_mode)
                for k in range(len(syn2)):
                    one = dec.decode_segments(syn2[k])
                    assert all(np.array_equal(a, b[k]) for a, b in zip(one, want)), (io_mode, k)


def test_rejected_option_does_not_stick(oracle):
    """qb_set_option validates through the launch planner; a value it rejects must leave the
    handle exactly as it was (the old value restored, plans rebuilt), so that later unrelated
    options and decodes still work."""
    from paper_2508_07879_b200 import codes
    g = codes.build_tanner_graph(codes.toy_code_3x6())
    cfg = DecoderConfig(max_iterations=10)
    syn = gf2.pack_bits(np.array([[1, 0, 1], [0, 1, 1]], dtype=np.uint8))
    with Decoder(g, cfg) as dec:
        want = dec.decode_batch_segments(syn)
        with pytest.raises(ValueError, match="regular kernel"):
            dec.set_option(0, 2)  # QB_OPT_KERNEL = regular kernels on a (4,2) toy graph
        assert dec.get_option(0) == 0
        dec.set_option(7, 0)      # an unrelated plan-affecting option still goes through
        dec.set_option(7, 1)
        got = dec.decode_batch_segments(syn)
        assert all(np.array_equal(a, b) for a, b in zip(got, want))
    code = codes.make_code("bb72")
    with Decoder(code, DecoderConfig()) as dec:
        with pytest.raises(ValueError):
            dec.set_option(5, 12)  # QB_OPT_BATCH_VARIANT out of range
        assert dec.get_option(5) != 12


GOLD_CODES = __import__("os").path.join(__import__("os").path.dirname(__import__("os").path.abspath(__file__)),
                                         "golden", "codes")


@pytest.mark.parametrize("mode", ["float", "int8", "int16"])
def test_codes_loaded_from_alist_and_json_files_decode_like_the_oracle(oracle, mode):
    """user-supplied matrices reach the degree-padded kernels through the
    on-disk formats.  Hand-written alist fixtures (the reference's own toy text, unpadded and
    zero-padded: proj/tests/test_alist.cpp:27-60), a committed irregular 40 x 70 matrix, and
    CSS-JSON descriptors (alist-file and bb constructions) are loaded, decoded in batch and
    compared with the oracle bit for bit."""
    import os
    from paper_2508_07879_b200 import alist, css_json
    rng = np.random.default_rng(17)
    toy = alist.load(os.path.join(GOLD_CODES, "toy_3x6.alist"))
    assert np.array_equal(toy.coo(), codes.toy_code_3x6().coo())
    assert np.array_equal(alist.load(os.path.join(GOLD_CODES, "toy_3x6_padded.alist")).coo(), toy.coo())
    irr = alist.load(os.path.join(GOLD_CODES, "irregular_40x70.alist"))
    for h, shots, iters in ((toy, 8, 10), (irr, 500, 25)):
        g = codes.build_tanner_graph(h)
        syn = (gf2.pack_bits(np.array([[(i >> b) & 1 for b in range(3)] for i in range(8)], dtype=np.uint8))
               if shots == 8 else random_syndromes(rng, shots, g.num_checks, 0.08))
        cfg = DecoderConfig(max_iterations=iters, arithmetic=mode)
        with Decoder(g, cfg) as dec:
            assert dec.get_option(OPT_INFO_ELL) != 0, "served by the degree-padded kernel"
            est, res, conv, its = dec.decode_batch_segments(syn)
        oe, ores, oc, oi = oracle.decode_many(g, cfg, syn)
        assert np.array_equal(est, oe) and np.array_equal(res, ores)
        assert np.array_equal(conv, oc) and np.array_equal(its, oi)
    # CSS codes from descriptors: files next to the JSON, and the bb construction
    for fname, want in (("bb72_files.json", "bb72"), ("bb144_bb.json", "bb144")):
        code = css_json.load(os.path.join(GOLD_CODES, fname))
        ref_code = codes.make_code(want)
        assert code.n == ref_code.n and code.k == ref_code.k
        from tests.helpers import error_syndromes
        _, _, syn = error_syndromes(code, rng, 200, 0.03)
        cfg = DecoderConfig(max_iterations=20, arithmetic=mode)
        with Decoder(code, cfg) as dec:
            est, res, conv, its = dec.decode_batch_segments(syn)
        oe, ores, oc, oi = oracle.decode_many(code.combined_graph, cfg, syn, code.segments)
        assert np.array_equal(est, oe) and np.array_equal(res, ores)
        assert np.array_equal(conv, oc) and np.array_equal(its, oi)
    # ... and the extended graph of a descriptor-loaded code goes through the (7,3) kernel
    code = css_json.load(os.path.join(GOLD_CODES, "bb72_files.json"))
    hext, segs = codes.extended_graph(code)
    ge = codes.build_tanner_graph(hext)
    syn = random_syndromes(rng, 300, ge.num_checks, 0.05)
    cfg = DecoderConfig(max_iterations=15, arithmetic=mode, priors=[3.0] * ge.num_vars)
    with Decoder(ge, cfg, segments=segs) as dec:
        assert dec.get_option(OPT_INFO_ELL) == 703
        est, res, conv, its = dec.decode_batch_segments(syn)
    oe, ores, oc, oi = oracle.decode_many(ge, cfg, syn, segs)
    assert np.array_equal(est, oe) and np.array_equal(its, oi)
