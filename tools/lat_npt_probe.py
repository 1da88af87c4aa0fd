"""Single-shot latency by nodes-per-thread shape of the cluster kernel (dev tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2508_07879_b200 import Decoder, DecoderConfig, codes, gf2
for name in ("bb784", "bb144"):
    code = codes.make_code(name)
    rng = np.random.default_rng(1)
    n = code.n
    ex = (rng.random((256, n)) < 0.01).astype(np.uint8); ez = (rng.random((256, n)) < 0.01).astype(np.uint8)
    pool = gf2.pack_bits(np.concatenate([code.hz.mat_vec(ex), code.hx.mat_vec(ez)], axis=-1))
    for arith in ("float", "half", "int8"):
        for iters, early in ((10, False), (50, True)):
            cfg = DecoderConfig(max_iterations=iters, early_termination=early, arithmetic=arith)
            with Decoder(code, cfg) as dec:
                ref = None
                for npt in (1, 2, 3):
                    try:
                        dec.set_option(6, npt)
                    except Exception as e:
                        print(name, arith, npt, "n/a", e); continue
                    for io in (2, 0):
                        dec.set_option(1, io)
                        w, k, dg = dec.latency_run(pool, 300, 3000)
                        ref = ref or dg
                        assert dg == ref, "digest differs"
                        print(name, arith, iters, int(early), "npt", npt, "io", io, "threads", dec.get_option(103) if False else "",
                              "p50 %.2f p99 %.2f kernel p50 %.2f" % (np.percentile(w, 50) / 1e3, np.percentile(w, 99) / 1e3, np.median(k) / 1e3), flush=True)
