import numpy as np, sys
sys.path.insert(0,'.')
from paper_2508_07879_b200 import Decoder, DecoderConfig, codes, gf2
code=codes.make_code("bb784")
hx,segs=codes.extended_graph(code); gx=codes.build_tanner_graph(hx)
rng=np.random.default_rng(1); pq=0.005
pool=gf2.pack_bits(hx.mat_vec((rng.random((256,gx.num_vars))<pq).astype(np.uint8)))
llr=np.abs(rng.standard_normal((256,gx.num_checks)))*5+0.5
for arith in ("int8","int16","float","half"):
    cfg=DecoderConfig(max_iterations=10,early_termination=False,arithmetic=arith,priors=[5.3]*gx.num_vars)
    with Decoder(gx,cfg,segments=segs) as dec:
        soft=dec.quantize_soft(llr)
        for io,gr in ((2,1),(0,1),(1,1),(1,0)):
            dec.set_option(1,io); dec.set_option(12,gr)
            for sp in (None,soft):
                w,k,_=dec.latency_run(pool,300,3000,soft_pool=sp)
                print(arith,io,gr,'soft' if sp is not None else 'hard', np.median(w)/1e3, np.median(k)/1e3, flush=True)
