"""Batched boosted greedy AED (pgpb_aed_greedy_step, beams.AEDGreedyDecoder)
vs the reference's aed_beam_boosted at beam 1 (decoding.py:502-587, R10).

Every row an utterance consumed is recorded and replayed, keyed by its token
prefix (acoustic.py:236-237), into the oracle's restatement with
beam_size=1: tokens, fp64 am / boost and the trace (including the eos step
and its bump) must be identical.  Also checked at the config-4 bench shape
and against the device beam decoder at beam 1."""

import numpy as np
import pytest

import bench_workloads as bw
import gen_inputs as gi
from conftest import product_table, res_tuple

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def _replay(out, B, max_len, eos, tab, lam, V, bump=True, which=None, rollback=False):
    for b in (range(B) if which is None else which):
        rows = {}
        res = out.nbest[b]
        toks = list(res.tokens)
        for lp, ln, ended in out.records:
            n = int(ln[b])
            if ended[b] or n >= max_len:
                continue
            rows[tuple(toks[:n])] = lp[b].copy()
        exp = orc.aed_beam(lambda p, n: rows[tuple(p)], tab, lam, 1, max_len, eos, V, eos_bump=bump,
                           rollback=rollback)
        g = res_tuple(res)
        e = exp[0]
        assert g["tokens"] == e["tokens"], b
        assert g["am"] == e["am"] and g["boost"] == e["boost"], b
        assert g["trace"] == [list(x) for x in e["trace"]], b


@pytest.mark.parametrize("lam,max_len,bump,rollback", [(1.0, 8, True, False), (2.5, 6, True, False),
                                                       (1.0, 8, False, False), (0.0, 7, True, False),
                                                       (1.0, 8, True, True)])
def test_aed_greedy_matches_reference_beam1_by_replay(lam, max_len, bump, rollback):
    import torch

    from paper_2508_07014_b200 import DecodeConfig
    from paper_2508_07014_b200.beams import AEDGreedyDecoder, TransformerAEDModel

    V, B = 40, 16
    tab = product_table(gi.phrase_corpus(np.random.default_rng(7), V, 120), V)
    model = TransformerAEDModel(V, d_model=32, n_layers=2, n_heads=2, d_ff=64, max_len=max_len + 1, seed=1,
                                eos_id=V - 1, eos_bias=-1.0, eos_ramp=0.5)
    mem = torch.randn((B, 10, 32), device="cuda", generator=torch.Generator("cuda").manual_seed(3))
    cfg = DecodeConfig(lam=lam, beam_size=1, eos_bump_enabled=bump, rollback=rollback)
    dec = AEDGreedyDecoder(model, tab, cfg, B, max_len=max_len, eos=V - 1, poll=1, use_graph=False)
    out = dec.decode(mem, record=True, want_trace=True)
    assert any(r.trace and r.trace[-1].token == V - 1 for r in out.nbest)  # some utterances end on eos
    _replay(out, B, max_len, V - 1, tab, lam, V, bump, rollback=rollback)


def test_aed_greedy_equals_device_beam_1_and_graphs():
    import torch

    from paper_2508_07014_b200 import DecodeConfig
    from paper_2508_07014_b200.beams import AEDBeamDecoder, AEDGreedyDecoder, TransformerAEDModel

    V, B, max_len = 64, 12, 9
    tab = product_table(gi.phrase_corpus(np.random.default_rng(8), V, 200), V)
    model = TransformerAEDModel(V, d_model=32, n_layers=2, n_heads=2, d_ff=64, max_len=max_len + 1, seed=2,
                                eos_id=V - 1, eos_bias=-2.0, eos_ramp=0.6)
    mem = torch.randn((B, 10, 32), device="cuda", generator=torch.Generator("cuda").manual_seed(4))
    cfg = DecodeConfig(lam=1.5, beam_size=1)
    beam = AEDBeamDecoder(model, tab, cfg, B, max_len=max_len, eos=V - 1, use_graph=False).decode(
        mem, want_trace=True).nbest
    g = AEDGreedyDecoder(model, tab, cfg, B, max_len=max_len, eos=V - 1)
    for _ in range(3):  # eager warm-up, capture, replay
        got = g.decode(mem, want_trace=True).nbest
        for x, y in zip(got, beam):
            assert res_tuple(x) == res_tuple(y[0])


def test_aed_greedy_replay_at_config4_shape():
    """Config 4's model, table (20K phrases, V=4096), batch and max_len;
    8 utterances replayed (the oracle's pure-Python V-loop bounds the count)."""
    import torch

    from paper_2508_07014_b200 import DecodeConfig
    from paper_2508_07014_b200.beams import AEDGreedyDecoder

    dev = torch.device("cuda", 0)
    model, tab, mem = bw.config4(dev)
    c = bw.C4
    V = tab.vocab_size
    dec = AEDGreedyDecoder(model, tab, DecodeConfig(lam=1.0, beam_size=1), c["B"], max_len=c["max_len"], eos=V - 1,
                           poll=1, use_graph=False)
    out = dec.decode(mem, record=True, want_trace=True)
    _replay(out, c["B"], c["max_len"], V - 1, tab, 1.0, V, which=range(0, c["B"], c["B"] // 8))
