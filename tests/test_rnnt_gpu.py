"""Label-looping RNN-T greedy (GPU) vs the reference frame-synchronous decoder.

The random-init networks run on the GPU; parity replays the exact log-prob
row each utterance consumed at each (frame, symbol) step into the oracle's
restatement of transducer_greedy_boosted (decoding.py:350-393), which must
request rows in the same order with the same (frame, last token) context
and produce identical tokens, traces and scores.
"""

import numpy as np
import pytest

import gen_inputs as gi
from conftest import product_table

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def _replay_check(o, B, lengths, tab, lam, cap, blank=0):
    n = o.num_out.cpu().numpy()
    tok, dl, st = o.tokens.cpu().numpy(), o.deltas.cpu().numpy(), o.states.cpu().numpy()
    am, bo = o.am.cpu().numpy(), o.boost.cpu().numpy()
    for b in range(B):
        rows = [(r[0][b], int(r[2][b]), int(r[3][b])) for r in o.records if r[1][b]]
        it = iter(rows)

        def step(last, t):
            lp, t0, l0 = next(it)
            assert t0 == t, (b, t0, t)
            assert l0 == (blank if last is None else last)
            return lp

        e = orc.transducer_greedy(step, int(lengths[b]), blank, tab, lam, cap)
        assert next(it, None) is None, "GPU consumed rows the reference did not request"
        k = int(n[b])
        assert [int(x) for x in tok[b, :k]] == e["tokens"]
        assert float(am[b]) == e["am"] and float(bo[b]) == e["boost"]
        assert [[int(x), float(y), int(z)] for x, y, z in zip(tok[b, :k], dl[b, :k], st[b, :k])] == \
            [list(x) for x in e["trace"]]


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("lam,cap", [(1.0, 5), (2.0, 2), (0.0, 3)])
def test_label_looping_matches_reference_by_replay(lam, cap, fused):
    """Fused iteration (joint hidden + log-softmax fused into the boosted
    step + LSTM cell kernels) and the framework iteration: every row's
    decisions replayed into the oracle from the log-probs it was decided on."""
    import torch

    from paper_2508_07014_b200 import DecodeConfig
    from paper_2508_07014_b200.rnnt import LabelLoopingDecoder, RNNTModel

    phrases, V = gi.corpus("p5k_v1024")
    tab = product_table(phrases, V)
    B, T = 12, 40
    model = RNNTModel(V, enc_dim=64, pred_dim=64, joint_dim=64, seed=3, blank_bias=1.0)
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    enc = torch.randn((B, T, 64), generator=g, device="cuda")
    lengths = np.random.default_rng(1).integers(1, T + 1, size=B)
    dec = LabelLoopingDecoder(model, tab, DecodeConfig(lam=lam, max_symbols_per_frame=cap), B, T, use_graph=False,
                              fused=fused)
    assert dec.fused == fused
    o = dec.decode(model.project_encoder(enc), torch.from_numpy(lengths), record=True)
    assert int(o.num_out.sum()) > 0
    _replay_check(o, B, lengths, tab, lam, cap)
    if fused:
        # the fused log-softmax matches torch's on the recorded rows' logits
        # up to fp32 rounding (each recorded row is normalised)
        lp = np.concatenate([r[0][r[1].astype(bool)] for r in o.records])
        s = np.log(np.exp(lp.astype(np.float64)).sum(-1))
        assert np.abs(s).max() < 1e-5


def test_graph_replay_equals_eager_and_boost_changes_output():
    import torch

    from paper_2508_07014_b200 import DecodeConfig
    from paper_2508_07014_b200.rnnt import LabelLoopingDecoder, RNNTModel

    phrases, V = gi.corpus("p20k_v1024")
    tab = product_table(phrases, V)
    B, T = 32, 60
    model = RNNTModel(V, enc_dim=128, pred_dim=128, joint_dim=128, seed=5, blank_bias=1.0)
    enc = torch.randn((B, T, 128), device="cuda", generator=torch.Generator(device="cuda").manual_seed(9))
    ep = model.project_encoder(enc)
    outs = {}
    for lam in (0.0, 1.0):
        cfg = DecodeConfig(lam=lam)
        eager = LabelLoopingDecoder(model, tab, cfg, B, T, use_graph=False).decode(ep)
        e = (eager.tokens.clone(), eager.num_out.clone(), eager.am.clone(), eager.boost.clone())
        graph = LabelLoopingDecoder(model, tab, cfg, B, T, use_graph=True).decode(ep)
        assert torch.equal(e[1], graph.num_out)
        assert torch.equal(e[0], graph.tokens) and torch.equal(e[2], graph.am) and torch.equal(e[3], graph.boost)
        outs[lam] = e
    assert not torch.equal(outs[0.0][0], outs[1.0][0]), "boosting never changed a token"
    assert float(outs[0.0][3].abs().max()) == 0.0


def _tdt_replay_check(o, B, lengths, tab, lam, cap, blank=0):
    n = o.num_out.cpu().numpy()
    tok, dl, st = o.tokens.cpu().numpy(), o.deltas.cpu().numpy(), o.states.cpu().numpy()
    am, bo = o.am.cpu().numpy(), o.boost.cpu().numpy()
    for b in range(B):
        rows = [(r[0][b], int(r[2][b]), int(r[3][b]), int(r[4][b])) for r in o.records if r[1][b]]
        it = iter(rows)

        def step(last, t):
            lp, t0, l0, d = next(it)
            assert t0 == t, (b, t0, t)
            assert l0 == (blank if last is None else last)
            return lp, d

        e = orc.transducer_greedy_tdt(step, int(lengths[b]), blank, tab, lam, cap)
        assert next(it, None) is None, "GPU consumed rows the restatement did not request"
        k = int(n[b])
        assert [int(x) for x in tok[b, :k]] == e["tokens"]
        assert float(am[b]) == e["am"] and float(bo[b]) == e["boost"]
        assert [[int(x), float(y), int(z)] for x, y, z in zip(tok[b, :k], dl[b, :k], st[b, :k])] == \
            [list(x) for x in e["trace"]]


@pytest.mark.parametrize("lam,cap,durs", [(1.0, 3, (0, 1, 2, 3, 4)), (2.0, 2, (0, 2, 5)), (0.0, 4, (1, 2)),
                                          (1.0, 2, (0,))])
def test_tdt_label_looping_matches_restatement_by_replay(lam, cap, durs):
    import torch

    from paper_2508_07014_b200 import DecodeConfig
    from paper_2508_07014_b200.rnnt import LabelLoopingDecoder, RNNTModel

    phrases, V = gi.corpus("p5k_v1024")
    tab = product_table(phrases, V)
    B, T = 12, 50
    model = RNNTModel(V, enc_dim=64, pred_dim=64, joint_dim=64, seed=4, blank_bias=1.0, durations=durs)
    enc = torch.randn((B, T, 64), generator=torch.Generator(device="cuda").manual_seed(8), device="cuda")
    lengths = np.random.default_rng(2).integers(1, T + 1, size=B)
    dec = LabelLoopingDecoder(model, tab, DecodeConfig(lam=lam, max_symbols_per_frame=cap), B, T, use_graph=False)
    o = dec.decode(model.project_encoder(enc), torch.from_numpy(lengths), record=True)
    assert int(o.num_out.sum()) > 0
    _tdt_replay_check(o, B, lengths, tab, lam, cap)
    # graph replay gives the same outputs
    g = LabelLoopingDecoder(model, tab, DecodeConfig(lam=lam, max_symbols_per_frame=cap), B, T, use_graph=True)
    og = g.decode(model.project_encoder(enc), torch.from_numpy(lengths))
    assert torch.equal(og.num_out, o.num_out) and torch.equal(og.am, o.am) and torch.equal(og.tokens, o.tokens)
