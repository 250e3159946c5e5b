"""One small invocation of every libpgpb kernel, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck; scripts/gpu_sanitize.sh).
Small tables and batches keep the instrumented run short; each result is
checked against the oracle so a sanitizer-clean run is also a correct one."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import gen_inputs as gi  # noqa: E402
from conftest import product_table  # noqa: E402

import paper_2508_07014_b200 as pb  # noqa: E402
from oracle import oracle as orc  # noqa: E402

rng = np.random.default_rng(0)
V = 256
tab = product_table(gi.phrase_corpus(np.random.default_rng(1), V, 300), V)
dev = torch.device("cuda", 0)
# advance (v6), chained advance, chain walk
st = rng.integers(0, tab.num_states, size=300).astype(np.int32)
r = pb.get_scores_batch(tab, st)
sc, nx = orc.score_batch(tab, st)
assert np.array_equal(r.next_states, nx)
toks = torch.from_numpy(rng.integers(0, V, size=(3, 300)).astype(np.int32)).to(dev)
pb.advance_steps(tab, torch.from_numpy(st).to(dev), toks)  # compact arrays (V <= 1024)
from paper_2508_07014_b200 import _lib  # noqa: E402

for lay in (1, 2, 3):  # ranked-bitmap, compact-array and blob chained kernels
    _lib.set_tuning("adv.compact", lay)
    pb.advance_steps(tab, torch.from_numpy(st).to(dev), toks)
_lib.set_tuning("adv.compact", 0)
from paper_2508_07014_b200.table import _advance_device  # noqa: E402

_advance_device(tab, torch.from_numpy(st).to(dev), check=True, out=None, chain=True)
# greedy CTC (phase A + walker), boosted and not, ragged
lps = np.stack([gi.random_emissions(rng, 70, V) for _ in range(6)])
lens = np.array([70, 1, 0, 33, 70, 12], np.int32)
for lam in (0.0, 1.0):
    out = pb.ctc_greedy_boosted_batch(lps, lens, tab, pb.DecodeConfig(lam=lam), blank_id=0)
    e = orc.ctc_greedy_decode(lps[0], 0, tab, lam)
    assert out[0].tokens == e["tokens"]
# reference-API beams (beam_topk) incl. a multi-pass k
em = pb.EmissionMatrix(gi.random_emissions(rng, 8, V), blank_id=0)
pb.ctc_beam_boosted(em, tab, pb.DecodeConfig(lam=1.0, beam_size=40))
rows, default = gi.random_transducer_rows(rng, V)
m = pb.TableStepModel(flavor="transducer", default_row=default, rows=rows)
pb.transducer_beam_boosted(m, 4, 0, tab, pb.DecodeConfig(lam=1.0, beam_size=4, max_symbols_per_frame=2))
arows, adef = gi.random_aed_rows(rng, V)
am = pb.TableStepModel(flavor="aed", default_row=adef, rows=arows, eos_id=V - 1)
pb.aed_beam_boosted(am, tab, pb.DecodeConfig(lam=1.0, beam_size=4), max_len=4)
# greedy transducer step (host StepModel) and label looping (fused)
pb.transducer_greedy_boosted(m, 6, 0, tab, pb.DecodeConfig(lam=1.0))
from paper_2508_07014_b200.beams import (AEDBeamDecoder, AEDGreedyDecoder, StatelessTransducerModel,  # noqa: E402
                                         TransducerBeamDecoder, TransformerAEDModel)
from paper_2508_07014_b200.rnnt import LabelLoopingDecoder, RNNTModel  # noqa: E402

model = RNNTModel(V, enc_dim=32, pred_dim=32, joint_dim=32, seed=1, blank_bias=1.0)
enc = model.project_encoder(torch.randn((4, 12, 32), device=dev))
LabelLoopingDecoder(model, tab, pb.DecodeConfig(lam=1.0), 4, 12, use_graph=False).decode(enc)
# device beams
sm = StatelessTransducerModel(V, enc_dim=32, pred_dim=32, joint_dim=32, seed=1, blank_bias=0.5)
TransducerBeamDecoder(sm, tab, pb.DecodeConfig(lam=1.0, beam_size=4, max_symbols_per_frame=2), 3, 6,
                      use_graph=False).decode(sm.project_encoder(torch.randn((3, 6, 32), device=dev)))
amodel = TransformerAEDModel(V, d_model=32, n_layers=1, n_heads=2, d_ff=64, max_len=6, seed=1, eos_id=V - 1,
                             eos_bias=-1.0, eos_ramp=0.5)
mem = torch.randn((3, 5, 32), device=dev)
AEDBeamDecoder(amodel, tab, pb.DecodeConfig(lam=1.0, beam_size=4), 3, max_len=5, eos=V - 1, use_graph=False).decode(mem)
AEDGreedyDecoder(amodel, tab, pb.DecodeConfig(lam=1.0, beam_size=1), 3, max_len=5, eos=V - 1,
                 use_graph=False).decode(mem)
# device CTC prefix beam (pgpb_ctc_beam), boosted and not, ragged lengths
from paper_2508_07014_b200.beams import ctc_beam_batch  # noqa: E402

lps = np.stack([gi.random_emissions(rng, 10, V) for _ in range(3)])
for lam in (1.0, 0.0):
    out = ctc_beam_batch(lps, np.array([10, 1, 6], np.int32), tab, pb.DecodeConfig(lam=lam, beam_size=4), blank_id=0)
    assert [h.tokens for h in out[0][1]] == [h["tokens"] for h in orc.ctc_beam(lps[0], 0, tab, lam, 4)]
# keyphrase hits on the device
from paper_2508_07014_b200.evaluation import keyphrase_hits_device  # noqa: E402

keyphrase_hits_device([["a", "b", "c"], ["b", "c"]], [["a", "b"], ["c"]], ["a b", "b c"])
torch.cuda.synchronize()
print("sanitize workload ok")
