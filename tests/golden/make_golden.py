#!/usr/bin/env python
"""Generates the committed golden vectors from the UNMODIFIED reference
(oracle/_ref/libqldpc_ref.so, compiled in place from /root/reference by
oracle/Makefile).  Run in the authoring container only:

    python tests/golden/make_golden.py

Every fixture is an .npz holding the inputs (graph arrays or code name, config,
packed syndromes) and the reference's outputs (estimate / residual words,
converged, iterations) so that the CPU oracle and the CUDA path can be pinned
on the GPU box, where /root/reference does not exist.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Ref  # noqa: E402
from paper_2508_07879_b200 import DecoderConfig, gf2  # noqa: E402
from tests.helpers import random_ldpc_matrix  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
MODES = ("float", "int8", "int16")


def save(name, **arrays):
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **arrays)
    print("wrote", name, {k: getattr(v, "shape", None) for k, v in arrays.items()})


def css_fixture(ref, code_name, p, shots, max_iter, early, seed):
    """Combined-graph decode of sample_error-derived syndromes (run_bench's pool recipe)."""
    rc = ref.code(code_name)
    pool, ex, ez = ref.syndrome_pool(rc, p, seed, shots, with_errors=True)
    out = {"syndromes": pool, "ex": ex, "ez": ez, "p": p, "seed": seed,
           "max_iterations": max_iter, "early": int(early)}
    for mode in MODES:
        cfg = DecoderConfig(max_iterations=max_iter, early_termination=early, arithmetic=mode)
        dec = ref.decoder(rc, cfg)
        est, res, conv, its = dec.decode_many(pool)
        # per-segment outcome through decode_css_into
        cx = np.zeros(shots, dtype=np.uint8); cz = np.zeros(shots, dtype=np.uint8)
        ix = np.zeros(shots, dtype=np.uint32); iz = np.zeros(shots, dtype=np.uint32)
        mz, mx = rc.rows_z, rc.rows_x
        sb = gf2.unpack_bits(pool, mz + mx)
        for i in range(shots):
            (_, _, c0, i0), (_, _, c1, i1) = dec.decode_css(
                gf2.pack_bits(sb[i, :mz]), mz, gf2.pack_bits(sb[i, mz:]), mx, rc.n)
            cx[i], cz[i], ix[i], iz[i] = c0, c1, i0, i1
        out.update({f"{mode}_estimate": est, f"{mode}_residual": res, f"{mode}_converged": conv,
                    f"{mode}_iterations": its, f"{mode}_conv_seg": np.stack([cx, cz], 1),
                    f"{mode}_iters_seg": np.stack([ix, iz], 1)})
    save(f"css_{code_name}_p{p}_{'early' if early else 'fixed'}{max_iter}", **out)


def graph_fixture(ref, name, graph, cfg_kwargs, syndromes):
    out = {"edge_var": graph.edge_var, "check_offsets": graph.check_offsets,
           "var_offsets": graph.var_offsets, "var_edges": graph.var_edges,
           "num_checks": graph.num_checks, "num_vars": graph.num_vars, "syndromes": syndromes}
    for k, v in cfg_kwargs.items():
        out["cfg_" + k] = np.asarray(v)
    for mode in MODES:
        kw = dict(cfg_kwargs)
        if mode != "float" and "priors" in kw and kw.get("quant_scale", 0) == 0:
            kw["quant_scale"] = 16.0
        cfg = DecoderConfig(arithmetic=mode, **kw)
        try:
            est, res, conv, its = ref.decoder(graph, cfg).decode_many(syndromes)
        except ValueError:
            continue
        out.update({f"{mode}_estimate": est, f"{mode}_residual": res,
                    f"{mode}_converged": conv, f"{mode}_iterations": its,
                    f"{mode}_quant_scale": kw.get("quant_scale", 0.0)})
    save(name, **out)


def soft_fixture(ref, code_name, shots, p, mu, sigma, seed):
    """Soft (noisy) syndromes on the extended graph diag([Hz | I], [Hx | I]): the reference
    has priors per Decoder only, so every shot is decoded by its own unmodified reference
    Decoder whose priors carry that shot's reliabilities (ref_decode_many_soft).  Stored:
    the syndromes, the reliabilities as doubles AND in each mode's stored form (what the
    CUDA library is handed), and the reference's outcomes per mode."""
    from paper_2508_07879_b200 import codes
    code = codes.make_code(code_name)
    h, _ = codes.extended_graph(code)
    g = codes.build_tanner_graph(h)
    n, mz, mx = code.n, code.hz.rows, code.hx.rows
    rng = np.random.default_rng(seed)
    data = np.zeros(g.num_vars, dtype=bool)
    data[:n] = True
    data[n + mz:2 * n + mz] = True
    err = ((rng.random((shots, g.num_vars)) < p) & data[None, :]).astype(np.uint8)
    lm = (1.0 - 2.0 * h.mat_vec(err)) * mu + sigma * rng.standard_normal((shots, g.num_checks))
    syn = gf2.pack_bits((lm < 0).astype(np.uint8))
    llr = 2.0 * mu * np.abs(lm) / sigma ** 2
    meas = np.concatenate([np.arange(n, n + mz), np.arange(2 * n + mz, 2 * n + mz + mx)]).astype(np.uint32)
    llr_d = float(np.log((1 - p) / p))
    rg = ref.graph_from_coo(h.rows, h.cols, h.coo())
    out = {"code": code_name, "syndromes": syn, "llr": llr, "soft_vars": meas, "p": p, "mu": mu,
           "sigma": sigma, "prior_data": llr_d, "max_iterations": 30}
    for mode, scale, kmax in (("float", 0.0, 0), ("int8", 8.0, 127), ("int16", 256.0, 32767)):
        if mode == "float":
            stored = llr.astype(np.float32)
            as_prior = stored.astype(np.float64)
        else:
            q = np.clip(np.floor(llr * scale + 0.5), 1, kmax)   # llround of a positive value, 0 -> 1
            stored = q.astype(np.int8 if mode == "int8" else np.int16)
            as_prior = q / scale
        cfg = DecoderConfig(max_iterations=30, arithmetic=mode, priors=[llr_d] * g.num_vars)
        est, res, conv, its = ref.decode_many_soft(rg, cfg, syn, meas, as_prior)
        out.update({f"{mode}_soft": stored, f"{mode}_estimate": est, f"{mode}_residual": res,
                    f"{mode}_converged": conv, f"{mode}_iterations": its})
    save(f"soft_{code_name}_p{p}", **out)


def main():
    ref = Ref()
    if "--soft-only" in sys.argv:
        soft_fixture(ref, "bb144", 96, 0.01, 1.0, 0.45, 20260823)
        return
    # 1. the reference's toy 3x6 fixture, every syndrome (test_decoder.cpp:269-294)
    toy = ref.toy_graph()
    all8 = np.stack([gf2.pack_bits(np.array([(m >> k) & 1 for k in range(3)], dtype=np.uint8))
                     for m in range(8)])
    graph_fixture(ref, "toy_uniform", toy, dict(max_iterations=10, alpha=0.8), all8)
    graph_fixture(ref, "toy_priors", toy,
                  dict(max_iterations=10, alpha=0.8, priors=[0.5, 1.25, 2.0, 0.75, 3.0, 1.5]), all8)
    graph_fixture(ref, "toy_saturating", toy,
                  dict(max_iterations=10, alpha=0.8, quant_scale=16.0,
                       priors=[20.0, 1.0, -2.0, 500.0, 0.25, 1.0]), all8)
    # 2. irregular graphs with degree-1 checks and variables (test_decoder.cpp:436-447)
    rng = np.random.default_rng(20260822)
    for k in range(3):
        h = random_ldpc_matrix(rng, 7 + k, 12 + 2 * k)
        g = ref.graph_from_coo(h.rows, h.cols, h.coo())
        syn = gf2.pack_bits((rng.random((16, h.rows)) < 0.3).astype(np.uint8))
        graph_fixture(ref, f"irregular_{k}", g,
                      dict(max_iterations=10, alpha=0.8, early_termination=bool(k % 2)), syn)
    # 3. CSS codes on the reference's own sampler streams
    css_fixture(ref, "bb72", 0.02, 64, 50, True, 1)
    css_fixture(ref, "bb144", 0.01, 64, 10, False, 1)
    css_fixture(ref, "bb784", 0.01, 48, 50, True, 1)
    css_fixture(ref, "bb784", 0.03, 32, 10, False, 12345)
    # 3b. soft syndromes: one reference Decoder per shot on [H | I]
    soft_fixture(ref, "bb144", 96, 0.01, 1.0, 0.45, 20260823)
    # 4. node-operation KATs evaluated by the reference itself
    q = np.array([2.0, -3.0, 1.5])
    save("node_ops",
         cn_a=ref.check_node_update(q, 0, 1.0), cn_b=ref.check_node_update(q, 1, 1.0),
         cn_c=ref.check_node_update(q, 0, 0.5),
         cn_zero=ref.check_node_update([0.0, -2.0], 0, 1.0),
         cn_deg1=np.array([ref.check_node_update([5.0], 0, 0.8)[0],
                           ref.check_node_update([5.0], 1, 0.8)[0]]),
         vn_a=ref.variable_node_update(1.0, [-1.5, 2.0]),
         vn_b=ref.variable_node_update(1.0, [7.0]),
         quant=np.array([ref.quantize_saturate(v, sc, lim) for v, sc, lim in
                         [(1.0, 8.0, 127), (0.5, 256.0, 32767), (100.0, 8.0, 127),
                          (-100.0, 8.0, 127), (0.44, 8.0, 127), (0.43, 8.0, 127),
                          (-0.4375, 8.0, 127), (0.0, 8.0, 127)]]))
    # 5. graph digests of every code the builder knows (reference build_bb_code / registry)
    from paper_2508_07879_b200 import codes
    import json
    digests = {}
    for name in codes.BUILTIN_SPECS:
        rc = ref.code(name)
        entry = {"n": rc.n, "k": rc.k}
        for which in ("x", "z", "combined"):
            rg = rc.graph(which)
            tg = codes.TannerGraph(rg.num_checks, rg.num_vars, rg.edge_var, rg.edge_check,
                                   rg.check_offsets, rg.var_offsets, rg.var_edges)
            entry[which] = tg.digest()
        digests[name] = entry
    with open(os.path.join(OUT, "graph_digests.json"), "w") as f:
        json.dump(digests, f, indent=1, sort_keys=True)
    print("wrote graph_digests.json")


if __name__ == "__main__":
    main()
