"""Tune the aligned config-3 model: unboosted/boosted tokens per frame for
(alpha, alpha_blank, beta, gamma) settings on 16 utterances."""
import sys
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import numpy as np, torch
import bench_workloads as bw, paper_2508_07014_b200 as pb
from paper_2508_07014_b200.beams import StatelessTransducerModel, TransducerBeamDecoder
dev = torch.device('cuda', 0)
c = bw.C3
tab, V = bw.table(c['corpus'])
phrases, _ = bw.gi.corpus(c['corpus'])
rng = np.random.default_rng(77)
B = 16
tpf = np.stack([bw.config3_targets(rng, V, c['T'], phrases) for _ in range(B)])
tgt = [[int(x) for x in row if x >= 0] for row in tpf]
for a, ab, be, ga in [(2.5, 1.5, 1.5, 1.0), (4, 2.5, 3, 1), (5, 3, 4, 1.5), (6, 3, 5, 2), (4, 3, 5, 1)]:
    m = StatelessTransducerModel(V, enc_dim=512, pred_dim=640, joint_dim=640, seed=3, blank_bias=0.0).align(be, ga)
    enc = m.aligned_frames(torch.from_numpy(tpf).to(dev), alpha=a, alpha_blank=ab)
    out = []
    for lam in (0.0, 1.0):
        dec = TransducerBeamDecoder(m, tab, pb.DecodeConfig(lam=lam, beam_size=4, max_symbols_per_frame=5), B, c['T'])
        dec.run(enc)
        best = dec.results()
        n = np.mean([len(nb[0].tokens) for nb in best])
        acc = np.mean([nb[0].tokens == t for nb, t in zip(best, tgt)])
        out.append((round(n / c['T'], 3), round(float(acc), 2)))
    print((a, ab, be, ga), 'unboosted tok/frame, exact', out[0], 'boosted', out[1], flush=True)
