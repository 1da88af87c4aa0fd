import sys, time
sys.path.insert(0,'.')
from paper_2508_07879_b200 import Decoder, DecoderConfig, codes
code=codes.make_code("bb784")
for _ in range(3):
    d=Decoder(code, DecoderConfig()); d.close()
print("---- fourth creation", file=sys.stderr, flush=True)
t=time.perf_counter(); d=Decoder(code, DecoderConfig()); print("total ms", (time.perf_counter()-t)*1e3, file=sys.stderr); 
t=time.perf_counter(); d.close(); print("close ms", (time.perf_counter()-t)*1e3, file=sys.stderr)
