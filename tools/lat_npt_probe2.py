import sys, os
sys.path.insert(0, '.')
import numpy as np
from paper_2508_07879_b200 import Decoder, DecoderConfig, codes, gf2
for name in ("bb144","bb72"):
    code = codes.make_code(name)
    rng = np.random.default_rng(1); n = code.n
    ex = (rng.random((256, n)) < 0.01).astype(np.uint8); ez = (rng.random((256, n)) < 0.01).astype(np.uint8)
    pool = gf2.pack_bits(np.concatenate([code.hz.mat_vec(ex), code.hx.mat_vec(ez)], axis=-1))
    for arith in ("float","int8"):
        cfg = DecoderConfig(max_iterations=10, early_termination=False, arithmetic=arith)
        for label, mk in (("one-cta", lambda: Decoder(code.combined_graph, cfg)), ("cluster", lambda: Decoder(code, cfg))):
            with mk() as dec:
                for npt in (1, 3):
                    dec.set_option(6, npt); dec.set_option(1, 2)
                    w, k, dg = dec.latency_run(pool, 300, 3000)
                    print(name, arith, label, "npt", npt, "p50 %.2f p99 %.2f kernel %.2f" % (np.percentile(w,50)/1e3, np.percentile(w,99)/1e3, np.median(k)/1e3), flush=True)
