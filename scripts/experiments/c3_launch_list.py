import sys
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import torch
import bench_workloads as bw, paper_2508_07014_b200 as pb
from paper_2508_07014_b200.beams import TransducerBeamDecoder
dev = torch.device('cuda', 0)
model, tab, enc = bw.config3(dev)
c = bw.C3
T = 20
dec = TransducerBeamDecoder(model, tab, pb.DecodeConfig(lam=1.0, beam_size=4, max_symbols_per_frame=5), c['B'], T, use_graph=False)
e = enc[:, :T].contiguous() if enc.dim() == 3 else enc
dec.run(e); torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
dec.run(e); torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
