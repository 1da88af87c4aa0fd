"""Throughput of the batch path on the extended (phenomenological) graph diag([Hz|I],[Hx|I]) - dev tool."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2508_07879_b200 import Decoder, DecoderConfig, codes, gf2, _lib
if os.environ.get("QB_LIB"):  # A/B runs of differently built libraries (dev only)
    _lib.LIB_PATH = os.path.abspath(os.environ["QB_LIB"])

ap = argparse.ArgumentParser()
ap.add_argument("--code", default="bb784")
ap.add_argument("--shots", type=int, default=1 << 17)
ap.add_argument("--p", type=float, default=0.01)
ap.add_argument("--q", type=float, default=0.01)
ap.add_argument("--ariths", default="int8,float,half")
ap.add_argument("--iters", default="50:1,10:0")
ap.add_argument("--kernel", type=int, default=0)
args = ap.parse_args()
code = codes.make_code(args.code)
h, segs = codes.extended_graph(code)
g = codes.build_tanner_graph(h)
n, mz, mx = code.n, code.hz.rows, code.hx.rows
llr_d, llr_m = np.log((1 - args.p) / args.p), np.log((1 - args.q) / args.q)
priors = np.concatenate([np.full(n, llr_d), np.full(mz, llr_m), np.full(n, llr_d), np.full(mx, llr_m)])
probs = np.concatenate([np.full(n, args.p), np.full(mz, args.q), np.full(n, args.p), np.full(mx, args.q)])
sw, ew = gf2.num_words(g.num_checks), gf2.num_words(g.num_vars)
dev = torch.device("cuda"); shots = args.shots
d_syn = torch.zeros((shots, sw), dtype=torch.int64, device=dev)
d_est = torch.zeros((shots, ew), dtype=torch.int64, device=dev)
d_conv = torch.zeros((shots, 2), dtype=torch.uint8, device=dev)
d_its = torch.zeros((shots, 2), dtype=torch.int32, device=dev)
stream = torch.cuda.current_stream().cuda_stream
for spec in args.iters.split(","):
    mi, early = spec.split(":")
    for arith in args.ariths.split(","):
        cfg = DecoderConfig(max_iterations=int(mi), early_termination=bool(int(early)), arithmetic=arith,
                            priors=priors.tolist())
        with Decoder(g, cfg, segments=segs) as dec:
            if args.kernel: dec.set_option(0, args.kernel)
            dec.generate_syndromes(1, 0.0, shots, d_syn.data_ptr(), None, probs=probs, css_interleave=False, stream=stream)
            f = lambda: dec.decode_batch_device(shots, d_syn.data_ptr(), d_est.data_ptr(), None, d_conv.data_ptr(), d_its.data_ptr(), stream)
            f(); f(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3): f()
            e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 3
            its = d_its.to(torch.int64)
            eu = float(its.sum()) * (g.num_edges // 2)
            print(json.dumps({"graph": "ext-" + args.code, "arith": arith, "max_iter": int(mi), "early": int(early),
                              "ctas_per_sm": dec.get_option(100), "block": dec.get_option(101),
                              "Mshots_s": shots / ms / 1e3, "G_edge_updates_s": eu / ms / 1e6,
                              "mean_iters": float(its.max(dim=1).values.double().mean()),
                              "conv": float(d_conv.min(dim=1).values.double().mean())}), flush=True)
