"""Throughput sweep over kernel variants (dev tool; numbers for DESIGN.md)."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2508_07879_b200 import Decoder, DecoderConfig, codes, gf2, _lib
if os.environ.get("QB_LIB"):  # A/B runs of differently built libraries (dev only)
    _lib.LIB_PATH = os.path.abspath(os.environ["QB_LIB"])

ap = argparse.ArgumentParser()
ap.add_argument("--code", default="bb784")
ap.add_argument("--shots", type=int, default=1 << 19)
ap.add_argument("--p", type=float, default=0.01)
ap.add_argument("--ariths", default="float,int8,half,int16")
ap.add_argument("--npts", default="1,2,3,4,5,6")
ap.add_argument("--ctas", default="0")
ap.add_argument("--iters", default="50:1,10:0")
ap.add_argument("--kernel", type=int, default=0)
ap.add_argument("--shapes", default="2")
ap.add_argument("--pairs", type=int, default=1)
ap.add_argument("--spread", default="1", help="QB_OPT_SLOT_SPREAD values to sweep")
ap.add_argument("--priors", type=int, default=0, help="1: per-variable LLR priors (general path)")
args = ap.parse_args()
code = codes.make_code(args.code)
g = code.combined_graph
sw, ew = gf2.num_words(g.num_checks), gf2.num_words(g.num_vars)
dev = torch.device("cuda")
shots = args.shots
d_syn = torch.zeros((shots, sw), dtype=torch.int64, device=dev)
d_est = torch.zeros((shots, ew), dtype=torch.int64, device=dev)
d_conv = torch.zeros((shots, 2), dtype=torch.uint8, device=dev)
d_its = torch.zeros((shots, 2), dtype=torch.int32, device=dev)
stream = torch.cuda.current_stream().cuda_stream
for spec in args.iters.split(","):
    mi, early = spec.split(":")
    for arith in args.ariths.split(","):
        pri = None
        if args.priors:
            pri = (np.log((1 - args.p) / args.p) * (1.0 + 0.1 * np.random.default_rng(5).random(g.num_vars))).tolist()
        cfg = DecoderConfig(max_iterations=int(mi), early_termination=bool(int(early)), arithmetic=arith, priors=pri)
        with Decoder(code, cfg) as dec:
            dec.generate_syndromes(1, args.p, shots, d_syn.data_ptr(), None, stream=stream)
            if args.kernel: dec.set_option(0, args.kernel)
            dec.set_option(10, args.pairs)
            for shape, npt in [(int(sh), int(x)) for sh in args.shapes.split(",") for x in args.npts.split(",")]:
              for spread in [int(x) for x in args.spread.split(",")]:
                for ctas in [int(x) for x in args.ctas.split(",")]:
                    dec.set_option(8, shape); dec.set_option(5, npt); dec.set_option(4, ctas)
                    dec.set_option(14, spread)
                    f = lambda: dec.decode_batch_device(shots, d_syn.data_ptr(), d_est.data_ptr(), None, d_conv.data_ptr(), d_its.data_ptr(), stream)
                    f(); f(); torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(); 
                    for _ in range(3): f()
                    e1.record(); torch.cuda.synchronize()
                    ms = e0.elapsed_time(e1) / 3
                    its = d_its.to(torch.int64)
                    eu = float((its.sum(dim=0) * torch.tensor([g.num_edges // 2] * 2, device=dev)).sum())
                    print(json.dumps({"arith": arith, "max_iter": int(mi), "early": int(early), "shape": shape, "npt": npt, "spread": spread,
                                      "ctas_req": ctas, "ctas_per_sm": dec.get_option(100), "block": dec.get_option(101),
                                      "Mshots_s": shots / ms / 1e3, "G_edge_updates_s": eu / ms / 1e6,
                                      "mean_iters": float(its.max(dim=1).values.double().mean()), "conv": float(d_conv.min(dim=1).values.double().mean())}), flush=True)
