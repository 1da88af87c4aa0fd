"""Throughput of the batch path on a random irregular graph (degree-padded kernels) - dev tool."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2508_07879_b200 import Decoder, DecoderConfig, codes, gf2, _lib
if os.environ.get("QB_LIB"):
    _lib.LIB_PATH = os.path.abspath(os.environ["QB_LIB"])
rng = np.random.default_rng(3)
rows, cols = 400, 800
dense = np.zeros((rows, cols), dtype=np.uint8)
for n in range(cols):                       # variable degrees 1..4
    for m in rng.choice(rows, size=int(rng.integers(1, 5)), replace=False):
        dense[m, n] = 1
dense = dense[:, :] 
for m in range(rows):                       # cap check degree at 12
    nz = np.nonzero(dense[m])[0]
    if len(nz) > 12: dense[m, nz[12:]] = 0
h = codes.SparseMatrix.from_dense(dense)
g = codes.build_tanner_graph(h)
shots = 1 << 17
syn = gf2.pack_bits((rng.random((shots, rows)) < 0.05).astype(np.uint8))
d_syn = torch.from_numpy(syn.view(np.int64)).cuda()
ew = gf2.num_words(cols)
d_est = torch.zeros((shots, ew), dtype=torch.int64, device="cuda")
d_conv = torch.zeros((shots, 1), dtype=torch.uint8, device="cuda"); d_its = torch.zeros((shots, 1), dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for arith in ("float", "int8", "half"):
    with Decoder(g, DecoderConfig(max_iterations=10, early_termination=False, arithmetic=arith)) as dec:
        f = lambda: dec.decode_batch_device(shots, d_syn.data_ptr(), d_est.data_ptr(), None, d_conv.data_ptr(), d_its.data_ptr(), st)
        f(); f(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); f(); f(); e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(json.dumps({"arith": arith, "ell": dec.get_option(107), "edges": g.num_edges, "Mshots_s": shots / ms / 1e3,
                          "G_edge_updates_s": shots * 10 * g.num_edges / ms / 1e6}))
