"""Distribution of the end-to-end batch call time (dev tool)."""
import sys, os, time, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2508_07879_b200 import Decoder, DecoderConfig, codes, gf2, _lib
lib = _lib.load()
code = codes.make_code("bb784"); g = code.combined_graph
shots = 1 << 20
sw, ew = gf2.num_words(g.num_checks), gf2.num_words(g.num_vars)
d_syn = torch.zeros((shots, sw), dtype=torch.int64, device="cuda")
def pinned(n):
    p = C.c_void_p(); assert lib.qb_host_alloc(C.byref(p), n) == 0; return p
h_syn, h_est, h_conv, h_its = pinned(shots*sw*8), pinned(shots*ew*8), pinned(shots*2), pinned(shots*8)
with Decoder(code, DecoderConfig(max_iterations=50)) as dec:
    dec.generate_syndromes(1, 0.01, shots, d_syn.data_ptr(), None, stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    host = d_syn.cpu().numpy(); C.memmove(h_syn, host.ctypes.data, shots*sw*8)
    for chunk in ([int(x) for x in sys.argv[1:]] or [0]):
        dec.set_option(15, chunk)
        ts = []
        for i in range(25):
            t0 = time.perf_counter(); dec.decode_batch_raw(shots, h_syn.value, h_est.value, None, h_conv.value, h_its.value); ts.append(time.perf_counter() - t0)
        ts = np.array(ts[3:]) * 1e3
        print("chunk", chunk, "ms min %.3f med %.3f max %.3f -> M/s med %.1f best %.1f" % (ts.min(), np.median(ts), ts.max(), shots/np.median(ts)/1e3, shots/ts.min()/1e3), flush=True)
