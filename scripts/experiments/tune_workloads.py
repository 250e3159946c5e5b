"""Emission-rate sweep for the synthetic config-3 / config-4 workloads.

Config 3 (RNN-T beam 4, stateless pred net): blank_bias vs tokens per frame
(target: config 2's ~0.3).  Config 4 (AED beam 4): eos bias / ramp vs the
best hypothesis length (target: hypotheses that end well inside max_len).
Prints one JSON line per setting."""
import json
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import gen_inputs as gi  # noqa: E402

import paper_2508_07014_b200 as pb  # noqa: E402
from paper_2508_07014_b200.beams import (AEDBeamDecoder, StatelessTransducerModel, TransducerBeamDecoder,  # noqa: E402
                                         TransformerAEDModel)


def table(name):
    phrases, V = gi.corpus(name)
    ctx = pb.ContextList([pb.Phrase(" ".join(map(str, p)), p) for p in phrases], min_chars=0)
    return pb.compile_arc_table(pb.compute_fail_links(pb.build_prefix_tree(ctx, pb.TreeParams(), V))), V


def timed(fn):
    fn()
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return statistics.median(ts)


dev = torch.device("cuda")
which = sys.argv[1] if len(sys.argv) > 1 else "both"
if which in ("3", "both"):
    tab5, V = table("p5k_v1024")
    B, T, D = 64, 200, 512
    g = torch.Generator(device=dev)
    g.manual_seed(77)
    raw = torch.randn((B, T, D), generator=g, device=dev)
    for bb in [float(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "4,2,1,0.5,0,-0.5,-1").split(",")]:
        model = StatelessTransducerModel(V, enc_dim=D, pred_dim=640, joint_dim=640, seed=3, blank_bias=bb)
        enc = model.project_encoder(raw)
        row = {"config": 3, "blank_bias": bb}
        for name, lam in (("unboosted", 0.0), ("boosted", 1.0)):
            dec = TransducerBeamDecoder(model, tab5, pb.DecodeConfig(lam=lam, beam_size=4, max_symbols_per_frame=5),
                                        B, T)
            ms = timed(lambda: dec.run(enc))
            best = dec.results()
            n = float(np.mean([len(nb[0].tokens) if nb else 0 for nb in best]))
            row[name] = {"ms": round(ms, 3), "tok_per_frame": round(n / T, 3), "waves": dec.launches}
        row["overhead"] = round(row["boosted"]["ms"] / row["unboosted"]["ms"] - 1, 4)
        print(json.dumps(row), flush=True)
if which in ("4", "both"):
    tab20, V4 = table("p20k_v4096")
    B, Tm, max_len = 64, 100, 48
    g = torch.Generator(device=dev)
    g.manual_seed(77)
    mem = torch.randn((B, Tm, 256), generator=g, device=dev)
    for spec in (sys.argv[3].split(";") if len(sys.argv) > 3 else ["0,0", "2,0.1", "0,0.3", "-2,0.3", "-4,0.4"]):
        bias, ramp = (float(x) for x in spec.split(","))
        model = TransformerAEDModel(V4, d_model=256, n_layers=4, n_heads=4, d_ff=1024, max_len=max_len + 1, seed=5,
                                    eos_id=V4 - 1, eos_bias=bias, eos_ramp=ramp)
        row = {"config": 4, "eos_bias": bias, "eos_ramp": ramp}
        for name, lam in (("unboosted", 0.0), ("boosted", 1.0)):
            dec = AEDBeamDecoder(model, tab20, pb.DecodeConfig(lam=lam, beam_size=4), B, max_len=max_len, eos=V4 - 1)
            ms = timed(lambda: dec.run(mem))
            best = dec.results()
            lens = [len(nb[0].tokens) if nb else 0 for nb in best]
            row[name] = {"ms": round(ms, 3), "len_mean": float(np.mean(lens)), "len_min": int(min(lens)),
                         "len_max": int(max(lens)), "steps": dec.launches}
        row["overhead"] = round(row["boosted"]["ms"] / row["unboosted"]["ms"] - 1, 4)
        print(json.dumps(row), flush=True)
