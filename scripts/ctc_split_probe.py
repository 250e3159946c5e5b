"""Upper bound of splitting each long utterance into S independently walked
segments: the reference corpus (25 x ~1803 frames) decoded as 25*S
utterances of ~1803/S frames (same frames, same bytes)."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
sys.path.insert(0, str(ROOT / "scripts"))
import ctc_regimes as cr  # noqa: E402
import gen_inputs as gi  # noqa: E402

import paper_2508_07014_b200 as pb  # noqa: E402
from paper_2508_07014_b200.acoustic import synth_ctc_emissions  # noqa: E402
from paper_2508_07014_b200.context import Vocabulary  # noqa: E402

tab, V = cr.table()
vocab = Vocabulary(tokens=tuple(str(i) for i in range(V)), blank_id=0)
targets, seeds, _ = gi.reference_overhead_corpus()
ems = [synth_ctc_emissions(tg, vocab, margin=0.5, seed=sd, boost_positions=[], blanks_between=3).logprobs
       for tg, sd in zip(targets, seeds)]
Tm = max(e.shape[0] for e in ems)
for S in (1, 2, 4, 8):
    L = -(-Tm // S)
    segs, lens = [], []
    for e in ems:
        for k in range(S):
            part = e[k * L:(k + 1) * L]
            pad = np.zeros((L, V), np.float32)
            pad[:part.shape[0]] = part
            segs.append(pad)
            lens.append(part.shape[0])
    lp = torch.from_numpy(np.stack(segs)).cuda()
    ln = torch.tensor(lens, dtype=torch.int32).cuda()
    r = [round(cr.timeit(lambda: pb.ctc_greedy_device(lp, ln, tab, pb.DecodeConfig(lam=l), 0)), 2) for l in (0.0, 1.0)]
    print("S", S, "utts", len(segs), "frames", L, r, "overhead", round(r[1] / r[0] - 1, 3), flush=True)
