"""Memcpy-protocol single-shot latency (dev tool): stream sync vs polling the copied record."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2508_07879_b200 import Decoder, DecoderConfig, codes, gf2
code = codes.make_code("bb784")
rng = np.random.default_rng(1); n = code.n
ex = (rng.random((256, n)) < 0.01).astype(np.uint8); ez = (rng.random((256, n)) < 0.01).astype(np.uint8)
pool = gf2.pack_bits(np.concatenate([code.hz.mat_vec(ex), code.hx.mat_vec(ez)], axis=-1))
cfg = DecoderConfig(max_iterations=10, early_termination=False)
with Decoder(code, cfg) as dec:
    for graph in (1, 0):
        dec.set_option(1, 1); dec.set_option(12, graph)
        for rep in range(3):
            w, k, dg = dec.latency_run(pool, 300, 5000)
            print("graph", graph, "p50 %.2f p99 %.2f mean %.2f digest %x" % (np.percentile(w, 50) / 1e3, np.percentile(w, 99) / 1e3, w.mean() / 1e3, dg), flush=True)
