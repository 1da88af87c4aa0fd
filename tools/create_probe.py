import time, sys
sys.path.insert(0,'.')
from paper_2508_07879_b200 import Decoder, DecoderConfig, codes
for name in ("bb72","bb784"):
    code=codes.make_code(name)
    for a in ("float","int8","int16","half"):
        ts=[]
        for i in range(6):
            t=time.perf_counter(); d=Decoder(code, DecoderConfig(arithmetic=a)); t1=time.perf_counter(); d.close(); ts.append((t1-t)*1e3)
        print(name,a,"create ms:", " ".join("%.1f"%x for x in ts), flush=True)
