#!/usr/bin/env python
"""BASELINE config 4: logical-error-rate sweep on [[784,24,24]] with the whole trial
loop on the GPU (qb_campaign_run), float / int8 / half, and - when the compiled
reference is available - the reference's run_campaign on a smaller trial count with
its 95 % binomial (Wilson) interval for comparison.  Prints one JSON line per point
and a markdown table (stdout)."""
import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_07879_b200 import DecoderConfig, codes  # noqa: E402
from paper_2508_07879_b200.campaign import Campaign, CampaignResult  # noqa: E402


def wilson(k, n, z=1.96):
    if n == 0:
        return 0.0, 1.0
    ph = k / n
    den = 1 + z * z / n
    c = (ph + z * z / (2 * n)) / den
    h = z * math.sqrt(ph * (1 - ph) / n + z * z / (4 * n * n)) / den
    return max(0.0, c - h), min(1.0, c + h)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--code", default="bb784")
    ap.add_argument("--trials", type=int, default=1 << 20)
    ap.add_argument("--ref-trials", type=int, default=20000)
    ap.add_argument("--ps", default="0.001,0.002,0.005,0.01,0.02,0.03,0.05")
    ap.add_argument("--modes", default="float,int8,half")
    ap.add_argument("--max-iterations", type=int, default=50)
    ap.add_argument("--seed", type=int, default=12345)
    ap.add_argument("--sampler", type=int, default=0,
                    help="QB_OPT_SAMPLER for the full-size runs: 0 = the reference's stream, 1 = "
                         "geometric skips (the runs on the reference's own trials always use 0)")
    args = ap.parse_args()
    code = codes.make_code(args.code)
    ref = rc = None
    try:
        from oracle.pyoracle import Ref
        if Ref.available() and args.ref_trials > 0:
            ref = Ref()
            rc = ref.code(args.code)
    except Exception:
        ref = None
    rows = []
    for mode in args.modes.split(","):
        camp = Campaign(code, DecoderConfig(max_iterations=args.max_iterations, arithmetic=mode))
        # untimed warm-up at the full chunk size: batch buffers, counters and the kernels'
        # lazy module load would otherwise be charged to the first point of the sweep
        camp.run_range(0.01, args.seed + 1, 0, args.trials)
        for p in [float(x) for x in args.ps.split(",")]:
            camp.decoder.set_option(16, args.sampler)
            t0 = time.perf_counter()
            r = CampaignResult.from_counters(camp.run_range(p, args.seed, 0, args.trials))
            dt = time.perf_counter() - t0
            camp.decoder.set_option(16, 0)
            fails = r.logical_x + r.logical_z + r.logical_both + r.non_converged
            row = {"code": args.code, "mode": mode, "p": p, "trials": r.trials, "ler": r.logical_error_rate,
                   "ler_ci95": wilson(fails, r.trials), "non_converged": r.non_converged,
                   "logical": r.logical_x + r.logical_z + r.logical_both,
                   "mean_iterations": r.mean_iterations, "trials_per_s": r.trials / dt}
            if ref is not None:
                rmode = "float" if mode == "half" else mode
                rr = ref.run_campaign(rc, 0, p, args.seed, args.ref_trials,
                                      DecoderConfig(max_iterations=args.max_iterations, arithmetic=rmode),
                                      workers=0)
                rf = rr["logical_x"] + rr["logical_z"] + rr["logical_both"] + rr["non_converged"]
                lo, hi = wilson(rf, args.ref_trials)
                glo, ghi = row["ler_ci95"]
                # the same trials on the GPU: bit-exact modes must reproduce the count itself
                same = CampaignResult.from_counters(camp.run_range(p, args.seed, 0, args.ref_trials))
                sf = same.logical_x + same.logical_z + same.logical_both + same.non_converged
                row.update(ref_mode=rmode, ref_trials=args.ref_trials, ref_ler=rr["logical_error_rate"],
                           ref_ci95=(lo, hi), gpu_ler_on_ref_trials=sf / args.ref_trials,
                           identical_on_ref_trials=bool(sf == rf) if mode != "half" else None,
                           within_ref_ci=bool(lo <= sf / args.ref_trials <= hi),
                           ci_overlap=bool(glo <= hi and lo <= ghi))
            rows.append(row)
            print(json.dumps(row), flush=True)
        camp.close()
    print("\n| mode | p | trials | LER (GPU) | mean it. | reference LER (trials) [95% CI] | GPU LER on the "
          "reference's trials | identical | within CI |")
    print("|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        refs = (f"{r['ref_ler']:.3e} ({r['ref_trials']}) [{r['ref_ci95'][0]:.2e}, {r['ref_ci95'][1]:.2e}]"
                if "ref_ler" in r else "-")
        print(f"| {r['mode']} | {r['p']} | {r['trials']} | {r['ler']:.3e} | {r['mean_iterations']:.2f} | "
              f"{refs} | {r.get('gpu_ler_on_ref_trials', float('nan')):.3e} | "
              f"{r.get('identical_on_ref_trials', '-')} | {r.get('within_ref_ci', '-')} |")
    print("\nThroughput of the whole loop (sample, syndrome, decode, classify on the device; host "
          "wall clock around qb_campaign_run, after one untimed warm-up run), M trials/s:\n")
    ps = sorted({r["p"] for r in rows})
    print("| mode | " + " | ".join(f"p = {p}" for p in ps) + " |")
    print("|---|" + "---|" * len(ps))
    for mode in args.modes.split(","):
        by_p = {r["p"]: r["trials_per_s"] for r in rows if r["mode"] == mode}
        print(f"| {mode} | " + " | ".join(f"{by_p[p] / 1e6:.1f}" if p in by_p else "-" for p in ps) + " |")


if __name__ == "__main__":
    main()
