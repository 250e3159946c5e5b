"""The synthetic decoder workloads of bench.py (BASELINE configs 2-4), built
in one place so the benchmark and the bench-shape parity tests
(tests/test_bench_shapes_gpu.py) decode exactly the same inputs.

Seeds, shapes and model settings are the bench's; `rank` shifts the seeds
per GPU under torchrun (each rank decodes its own utterances)."""

from __future__ import annotations

from functools import lru_cache

import numpy as np

import gen_inputs as gi

C2 = dict(B=128, T=200, D=512, pred=640, joint=640, blank_bias=10.5, corpus="p20k_v1024")
C3 = dict(B=64, T=200, D=512, pred=640, joint=640, beam=4, cap=5, corpus="p5k_v1024")
C4 = dict(B=64, Tm=100, d=256, layers=4, heads=4, ff=1024, max_len=48, beam=4, eos_bias=-4.0, eos_ramp=0.4,
          corpus="p20k_v4096")


@lru_cache(maxsize=4)
def table(name: str):
    import paper_2508_07014_b200 as pb

    phrases, V = gi.corpus(name)
    ctx = pb.ContextList([pb.Phrase(" ".join(map(str, p)), p) for p in phrases], min_chars=0)
    return pb.compile_arc_table(pb.compute_fail_links(pb.build_prefix_tree(ctx, pb.TreeParams(), V))), V


def config2(dev, rank: int = 0):
    """Greedy RNN-T label looping: LSTM-640 pred net + joint, 20K tree,
    128 x 200 frames.  Returns (model, table, enc_proj)."""
    import torch

    from paper_2508_07014_b200.rnnt import RNNTModel

    c = C2
    tab, V = table(c["corpus"])
    model = RNNTModel(V, enc_dim=c["D"], pred_dim=c["pred"], joint_dim=c["joint"], seed=11 + rank,
                      blank_bias=c["blank_bias"])
    g = torch.Generator(device=dev)
    g.manual_seed(4321 + rank)
    enc_proj = model.project_encoder(torch.randn((c["B"], c["T"], c["D"]), generator=g, device=dev))
    return model, tab, enc_proj


def config3_targets(rng, V, T, phrases, emit_rate=0.3, phrase_frac=0.6):
    """Per-frame targets of one synthetic utterance: about emit_rate of the
    frames carry a token (config 2's 0.3 tokens per frame), the rest are
    blank (-1); the token stream is a mix of key phrases from the tree's
    corpus (phrase_frac of the tokens) and random filler, so boosted beams
    walk deep tree states."""
    n = int(round(emit_rate * T))
    toks = []
    while len(toks) < n:
        if rng.random() < phrase_frac:
            toks.extend(int(x) for x in phrases[int(rng.integers(len(phrases)))])
        else:
            toks.extend(int(x) for x in rng.integers(1, V, size=int(rng.integers(1, 4))))
    toks = toks[:n]
    frames = np.full(T, -1, np.int64)
    pos = np.sort(rng.choice(T, size=n, replace=False))
    frames[pos] = toks
    return frames


def config3(dev, rank: int = 0):
    """RNN-T beam 4: stateless pred net + joint (random init, aligned
    structure: StatelessTransducerModel.align), 5K tree, 64 x 200 frames of
    synthetic projected encoder output with ~0.3 tokens per frame drawn from
    the tree's key phrases and filler (config3_targets)."""
    import numpy as np
    import torch

    from paper_2508_07014_b200.beams import StatelessTransducerModel

    c = C3
    tab, V = table(c["corpus"])
    phrases, _ = gi.corpus(c["corpus"])
    model = StatelessTransducerModel(V, enc_dim=c["D"], pred_dim=c["pred"], joint_dim=c["joint"], seed=3 + rank,
                                     blank_bias=0.0).align()
    rng = np.random.default_rng(77 + rank)
    tpf = np.stack([config3_targets(rng, V, c["T"], phrases) for _ in range(c["B"])])
    g = torch.Generator(device=dev)
    g.manual_seed(77 + rank)
    enc_proj = model.aligned_frames(torch.from_numpy(tpf).to(dev), generator=g)
    return model, tab, enc_proj


def config4(dev, rank: int = 0):
    """AED beam 4: 4-layer transformer decoder d=256, 20K tree at V=4096,
    batch 64, max_len 48; eos logit offset so hypotheses end inside max_len."""
    import torch

    from paper_2508_07014_b200.beams import TransformerAEDModel

    c = C4
    tab, V = table(c["corpus"])
    model = TransformerAEDModel(V, d_model=c["d"], n_layers=c["layers"], n_heads=c["heads"], d_ff=c["ff"],
                                max_len=c["max_len"] + 1, seed=5 + rank, eos_id=V - 1, eos_bias=c["eos_bias"],
                                eos_ramp=c["eos_ramp"])
    g = torch.Generator(device=dev)
    g.manual_seed(77 + rank)
    mem = torch.randn((c["B"], c["Tm"], c["d"]), generator=g, device=dev)
    return model, tab, mem
