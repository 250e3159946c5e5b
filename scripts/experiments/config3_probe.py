import sys, time
sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import numpy as np, torch
import bench_workloads as bw, paper_2508_07014_b200 as pb
from paper_2508_07014_b200.beams import TransducerBeamDecoder
dev=torch.device('cuda',0)
model, tab, enc = bw.config3(dev)
c=bw.C3
for lam in (0.0,1.0):
    dec=TransducerBeamDecoder(model, tab, pb.DecodeConfig(lam=lam, beam_size=4, max_symbols_per_frame=5), c['B'], c['T'])
    dec.run(enc); torch.cuda.synchronize()
    s,e=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    s.record(); dec.run(enc); e.record(); torch.cuda.synchronize()
    best=dec.results(want_trace=True)
    n=np.mean([len(nb[0].tokens) for nb in best]); deep=np.mean([sum(1 for st in nb[0].trace if st.boost>1.5) for nb in best])
    print('lam',lam,'ms',round(s.elapsed_time(e),2),'tok/frame',round(n/c['T'],3),'deep arcs/utt',round(deep,2), 'boost', round(float(np.mean([nb[0].boost_score for nb in best])),2))
