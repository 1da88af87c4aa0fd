"""Stage timing of the device campaign (sample+syndrome / decode / classify) - dev tool."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2508_07879_b200 import DecoderConfig, codes, gf2, _lib
if os.environ.get("QB_LIB"):
    _lib.LIB_PATH = os.path.abspath(os.environ["QB_LIB"])
from paper_2508_07879_b200.campaign import Campaign
code = codes.make_code("bb784"); g = code.combined_graph
shots = 1 << 20
SAMPLER = int(os.environ.get("QB_SAMPLER", "0"))  # 1 = geometric-skip sampler (QB_OPT_SAMPLER)
for arith in sys.argv[1:] or ["float"]:
    camp = Campaign(code, DecoderConfig(max_iterations=50, arithmetic=arith)); dec = camp.decoder
    dec.set_option(_lib.OPT_SAMPLER, SAMPLER)
    dec.set_option(15, int(os.environ.get("QB_CHUNK", "0")))  # trials per campaign round, 0 = default
    sw, ew = gf2.num_words(g.num_checks), gf2.num_words(g.num_vars)
    dev = torch.device("cuda")
    d_syn = torch.zeros((shots, sw), dtype=torch.int64, device=dev); d_err = torch.zeros((shots, ew), dtype=torch.int64, device=dev)
    d_est = torch.zeros((shots, ew), dtype=torch.int64, device=dev)
    d_conv = torch.zeros((shots, 2), dtype=torch.uint8, device=dev); d_its = torch.zeros((shots, 2), dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    def t(f, n=3):
        f(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n): f()
        e1.record(); torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n
    gen = t(lambda: dec.generate_syndromes(1, 0.01, shots, d_syn.data_ptr(), d_err.data_ptr(), stream=st))
    decd = t(lambda: dec.decode_batch_device(shots, d_syn.data_ptr(), d_est.data_ptr(), None, d_conv.data_ptr(), d_its.data_ptr(), st))
    cls = t(lambda: camp.classify_device(shots, d_err.data_ptr(), d_est.data_ptr(), d_syn.data_ptr(), d_conv.data_ptr(), d_its.data_ptr(), st))
    import time
    t0 = time.perf_counter(); c = camp.run_range(0.01, 1, 0, shots); whole = (time.perf_counter() - t0) * 1e3
    t0 = time.perf_counter(); c = camp.run_range(0.01, 1, 0, shots); whole = (time.perf_counter() - t0) * 1e3
    print(json.dumps({"arith": arith, "sampler": SAMPLER, "chunk": int(os.environ.get("QB_CHUNK", "0")), "generate_ms": gen, "decode_ms": decd, "classify_ms": cls, "campaign_ms": whole,
                      "campaign_Mtrials_s": shots / whole / 1e3}))
    camp.close()
