import sys, time
sys.path.insert(0,'.')
import torch, numpy as np
from paper_2508_07879_b200 import Decoder, DecoderConfig, codes, gf2
names=("bb72","bb144","bb784","bb756")
cs=[codes.make_code(n) for n in names]
torch.cuda.init()
def free(): 
    torch.cuda.synchronize(); return torch.cuda.mem_get_info()[0]
d=Decoder(cs[0], DecoderConfig()); d.close()
f0=free(); t=time.perf_counter()
N=int(sys.argv[1]) if len(sys.argv)>1 else 600
for i in range(N):
    c=cs[i%4]
    with Decoder(c, DecoderConfig(arithmetic=("float","int8","int16","half")[(i//4)%4])) as dec:
        syn=np.zeros((4, gf2.num_words(c.combined_graph.num_checks)),dtype=np.uint64)
        dec.decode_batch_segments(syn); dec.decode_segments(syn[0])
        if i%50==0: dec.set_option(1,2); dec.decode_segments(syn[0])
print(N, "cycles;", "create/decode/destroy cycles: %.1f s, device memory delta %.1f MB" % (time.perf_counter()-t, (f0-free())/1e6))
