#!/usr/bin/env python
"""BASELINE config 5: phenomenological noise on [[784,24,24]] - data flips p, measurement
flips q = p - decoded on the extended graph diag([Hz | I], [Hx | I]) with LLR priors and
int8-quantised messages.  The reference has no such noise model; its decoder
handles the graph through its generic path, so the comparison is the strongest possible one:
on the SAME (H, priors, syndromes) every outcome of the GPU decoder must equal the compiled
reference's, and the failure rate follows.

A shot FAILS if the decoder does not converge, if the corrected data error still has a
non-zero syndrome (the decoder blamed / missed a measurement error), or if it is a
non-trivial logical operator (overlap test with the code's logical operators, as the
device classifier of the campaign does).  Prints one JSON line per point and a markdown
table."""
import argparse
import json
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2508_07879_b200 import Decoder, DecoderConfig, codes, gf2  # noqa: E402
from paper_2508_07879_b200.campaign import residual_tests  # noqa: E402


def wilson(k, n, z=1.96):
    if n == 0:
        return 0.0, 1.0
    ph = k / n
    den = 1 + z * z / n
    c = (ph + z * z / (2 * n)) / den
    hw = z * math.sqrt(ph * (1 - ph) / n + z * z / (4 * n * n)) / den
    return max(0.0, c - hw), min(1.0, c + hw)


def failures(code, hz, hx, err_bits, est_bits, conv, tests_x, tests_z):
    """Per-shot failure flags from data errors / estimates in the extended layout."""
    n, mz = code.n, code.hz.rows
    ex, ez = err_bits[:, :n], err_bits[:, n + mz:2 * n + mz]
    hx_, hz_ = est_bits[:, :n], est_bits[:, n + mz:2 * n + mz]
    rx, rz = ex ^ hx_, ez ^ hz_
    bad = ~(conv.min(axis=1) == 1)
    bad |= hz.mat_vec(rx).any(axis=1) | hx.mat_vec(rz).any(axis=1)
    bad |= ((rx.astype(np.int32) @ tests_x.T.astype(np.int32)) & 1).any(axis=1)
    bad |= ((rz.astype(np.int32) @ tests_z.T.astype(np.int32)) & 1).any(axis=1)
    return bad


def main_soft(args):
    """Config 5 as named.  sigma is chosen per point so that a measured bit flips with
    probability p (mu = 1): sigma = 1 / Phi^-1(1 - p)."""
    from statistics import NormalDist
    code = codes.make_code(args.code)
    h, segs = codes.extended_graph(code)
    g = codes.build_tanner_graph(h)
    n, mz, mx = code.n, code.hz.rows, code.hx.rows
    tx, tz = residual_tests(code)
    tests_x = gf2.unpack_bits(tx, 2 * n)[:, :n]
    tests_z = gf2.unpack_bits(tz, 2 * n)[:, n:]
    from oracle.pyoracle import Ref
    ref = Ref() if Ref.available() else None
    rg = ref.graph_from_coo(h.rows, h.cols, h.coo()) if ref else None
    sw, ew = gf2.num_words(g.num_checks), gf2.num_words(g.num_vars)
    dev = torch.device("cuda")
    shots = args.trials
    sdt = torch.int8 if args.arithmetic == "int8" else torch.int16 if args.arithmetic == "int16" else torch.float32
    d_syn = torch.zeros((shots, sw), dtype=torch.int64, device=dev)
    d_err = torch.zeros((shots, ew), dtype=torch.int64, device=dev)
    d_est = torch.zeros((shots, ew), dtype=torch.int64, device=dev)
    d_soft = torch.zeros((shots, g.num_checks), dtype=sdt, device=dev)
    d_conv = torch.zeros((shots, 1), dtype=torch.uint8, device=dev)
    d_its = torch.zeros((shots, 1), dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    rows = []
    for p in [float(x) for x in args.ps.split(",")]:
        mu, sigma = 1.0, 1.0 / NormalDist().inv_cdf(1 - p)
        llr = float(np.log((1 - p) / p))
        cfg = DecoderConfig(max_iterations=args.max_iterations, arithmetic=args.arithmetic,
                            priors=[llr] * g.num_vars)
        with Decoder(g, cfg) as dec:   # ONE segment, as the reference's graph constructor
            dec.generate_soft_syndromes(args.seed, p, mu, sigma, shots, d_syn.data_ptr(),
                                        d_soft.data_ptr(), d_err.data_ptr(), stream=st)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dec.decode_batch_soft_device(shots, d_syn.data_ptr(), d_soft.data_ptr(), d_est.data_ptr(),
                                         None, d_conv.data_ptr(), d_its.data_ptr(), st)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            sv = dec.soft_vars()
            scale = cfg.quant_scale or (8.0 if args.arithmetic == "int8" else 256.0)
            err = gf2.unpack_bits(d_err.cpu().numpy().view(np.uint64), g.num_vars)
            est = gf2.unpack_bits(d_est.cpu().numpy().view(np.uint64), g.num_vars)
            conv = d_conv.cpu().numpy()
            its = d_its.cpu().numpy()
            bad = failures(code, code.hz, code.hx, err, est, conv, tests_x, tests_z)
            # hard-decision decoding of the same shots
            dec.decode_batch_device(shots, d_syn.data_ptr(), d_est.data_ptr(), None,
                                    d_conv.data_ptr(), d_its.data_ptr(), st)
            torch.cuda.synchronize()
            est_h = gf2.unpack_bits(d_est.cpu().numpy().view(np.uint64), g.num_vars)
            bad_h = failures(code, code.hz, code.hx, err, est_h, d_conv.cpu().numpy(), tests_x, tests_z)
            k = int(bad.sum())
            row = {"p": p, "sigma": sigma, "trials": shots, "failures": k, "ler": k / shots,
                   "ler_ci95": wilson(k, shots), "ler_hard_same_shots": float(bad_h.mean()),
                   "non_converged": int((conv.min(axis=1) == 0).sum()),
                   "mean_iterations": float(its.max(axis=1).mean()), "decodes_per_s": shots / ms * 1e3}
            if ref is not None:
                m = min(args.ref_trials, shots)
                syn_h = d_syn[:m].cpu().numpy().view(np.uint64)
                soft_h = d_soft[:m].cpu().numpy()
                dq = soft_h.astype(np.float64) / (1.0 if args.arithmetic == "float" else scale)
                rest, rres, rconv, rits = ref.decode_many_soft(rg, cfg, syn_h, sv, dq)
                same = bool(np.array_equal(gf2.pack_bits(est[:m]), rest)
                            and np.array_equal(conv[:m, 0], rconv) and np.array_equal(its[:m, 0], rits))
                rbits = gf2.unpack_bits(rest, g.num_vars)
                rbad = failures(code, code.hz, code.hx, err[:m], rbits, np.stack([rconv, rconv], axis=1),
                                tests_x, tests_z)
                row.update({"ref_trials": m, "ref_ler": float(rbad.mean()),
                            "ref_ci95": wilson(int(rbad.sum()), m),
                            "gpu_ler_on_ref_trials": float(bad[:m].mean()), "identical_to_reference": same})
        rows.append(row)
        print(json.dumps(row), flush=True)
    print()
    print("| p (data) = P(flip) | sigma | trials | LER soft (GPU) | 95% CI | LER hard, same shots | non-converged | "
          "mean it. | M decodes/s | reference (one Decoder per shot) LER [95% CI] | GPU on the same trials | "
          "outcomes identical |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        refcol = ("%.3e (%d) [%.2e, %.2e] | %.3e | %s" % (
            r["ref_ler"], r["ref_trials"], r["ref_ci95"][0], r["ref_ci95"][1],
            r["gpu_ler_on_ref_trials"], r["identical_to_reference"])) if "ref_ler" in r else "n/a | n/a | n/a"
        print("| %g | %.4f | %d | %.3e | [%.2e, %.2e] | %.3e | %d | %.2f | %.1f | %s |" % (
            r["p"], r["sigma"], r["trials"], r["ler"], r["ler_ci95"][0], r["ler_ci95"][1],
            r["ler_hard_same_shots"], r["non_converged"], r["mean_iterations"],
            r["decodes_per_s"] / 1e6, refcol))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--code", default="bb784")
    ap.add_argument("--trials", type=int, default=1 << 17)
    ap.add_argument("--ref-trials", type=int, default=2000)
    ap.add_argument("--ps", default="0.0005,0.001,0.002,0.003,0.005,0.0075,0.01")
    ap.add_argument("--max-iterations", type=int, default=50)
    ap.add_argument("--seed", type=int, default=2508)
    ap.add_argument("--soft", action="store_true",
                    help="soft (noisy) syndromes: Gaussian measurement channel with flip probability p, "
                         "per-shot priors through qb_decode_batch_soft; the reference arm builds one "
                         "Decoder per shot")
    ap.add_argument("--arithmetic", default="int8")
    args = ap.parse_args()
    if args.soft:
        return main_soft(args)
    code = codes.make_code(args.code)
    h, segs = codes.extended_graph(code)
    g = codes.build_tanner_graph(h)
    n, mz, mx = code.n, code.hz.rows, code.hx.rows
    tx, tz = residual_tests(code)
    tests_x = gf2.unpack_bits(tx, 2 * n)[:, :n]
    tests_z = gf2.unpack_bits(tz, 2 * n)[:, n:]
    ref = None
    try:
        from oracle.pyoracle import Ref
        if Ref.available():
            ref = Ref()
            rg = ref.graph_from_coo(h.rows, h.cols, h.coo())
    except Exception:
        ref = None
    sw, ew = gf2.num_words(g.num_checks), gf2.num_words(g.num_vars)
    dev = torch.device("cuda")
    shots = args.trials
    d_syn = torch.zeros((shots, sw), dtype=torch.int64, device=dev)
    d_err = torch.zeros((shots, ew), dtype=torch.int64, device=dev)
    d_est = torch.zeros((shots, ew), dtype=torch.int64, device=dev)
    d_conv = torch.zeros((shots, 1), dtype=torch.uint8, device=dev)
    d_its = torch.zeros((shots, 1), dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    rows = []
    for p in [float(x) for x in args.ps.split(",")]:
        llr = float(np.log((1 - p) / p))
        cfg = DecoderConfig(max_iterations=args.max_iterations, arithmetic="int8",
                            priors=[llr] * g.num_vars)
        # ONE segment, as the reference's graph constructor makes it (decoder.cpp:406-413: the
        # X and Z halves stop together), so the large-sample rate is the reference's own
        with Decoder(g, cfg) as dec:
            dec.generate_syndromes(args.seed, 0.0, shots, d_syn.data_ptr(), d_err.data_ptr(),
                                   probs=np.full(g.num_vars, p), css_interleave=False, stream=st)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dec.decode_batch_device(shots, d_syn.data_ptr(), d_est.data_ptr(), None,
                                    d_conv.data_ptr(), d_its.data_ptr(), st)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            kernel = "decode_ell_h2_kernel" if dec.get_option(10) else "decode_ell_kernel"
        err = gf2.unpack_bits(d_err.cpu().numpy().view(np.uint64), g.num_vars)
        est = gf2.unpack_bits(d_est.cpu().numpy().view(np.uint64), g.num_vars)
        conv = d_conv.cpu().numpy()
        its = d_its.cpu().numpy()
        bad = failures(code, code.hz, code.hx, err, est, conv, tests_x, tests_z)
        k = int(bad.sum())
        row = {"p": p, "q": p, "trials": shots, "failures": k, "ler": k / shots,
               "ler_ci95": wilson(k, shots), "non_converged": int((conv.min(axis=1) == 0).sum()),
               "mean_iterations": float(its.max(axis=1).mean()), "decodes_per_s": shots / ms * 1e3,
               "kernel": kernel}
        if ref is not None:
            m = min(args.ref_trials, shots)
            syn_h = d_syn[:m].cpu().numpy().view(np.uint64)
            # the reference's graph constructor makes ONE segment: decode that way on both sides
            rest, rres, rconv, rits = ref.decoder(rg, cfg).decode_many(syn_h)
            with Decoder(g, cfg) as dec1:
                gest, gres, gconv, gits = dec1.decode_batch_segments(syn_h)
            same = bool(np.array_equal(gest, rest) and np.array_equal(gres, rres)
                        and np.array_equal(gconv[:, 0], rconv) and np.array_equal(gits[:, 0], rits))
            rbits = gf2.unpack_bits(rest, g.num_vars)
            rconv2 = np.stack([rconv, rconv], axis=1)
            rbad = failures(code, code.hz, code.hx, err[:m], rbits, rconv2, tests_x, tests_z)
            gbits = gf2.unpack_bits(gest, g.num_vars)
            gconv2 = np.stack([gconv[:, 0], gconv[:, 0]], axis=1)
            gbad = failures(code, code.hz, code.hx, err[:m], gbits, gconv2, tests_x, tests_z)
            row.update({"ref_trials": m, "ref_ler": float(rbad.mean()), "ref_ci95": wilson(int(rbad.sum()), m),
                        "gpu_ler_on_ref_trials": float(gbad.mean()), "identical_to_reference": same})
        rows.append(row)
        print(json.dumps(row), flush=True)
    print()
    print("| p = q | trials | LER (GPU) | 95% CI | non-converged | mean it. | M decodes/s | "
          "reference LER [95% CI] | GPU on the same trials | outcomes identical |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        refcol = ("%.3e (%d) [%.2e, %.2e] | %.3e | %s" % (
            r["ref_ler"], r["ref_trials"], r["ref_ci95"][0], r["ref_ci95"][1],
            r["gpu_ler_on_ref_trials"], r["identical_to_reference"])) if "ref_ler" in r else "n/a | n/a | n/a"
        print("| %g | %d | %.3e | [%.2e, %.2e] | %d | %.2f | %.1f | %s |" % (
            r["p"], r["trials"], r["ler"], r["ler_ci95"][0], r["ler_ci95"][1], r["non_converged"],
            r["mean_iterations"], r["decodes_per_s"] / 1e6, refcol))


if __name__ == "__main__":
    main()
