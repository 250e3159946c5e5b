"""Device-resident batched beam search (beams.py, csrc/pgpb_dbeam.cu) vs the reference decoders.

The random-init networks run on the GPU; parity replays the exact log-prob
rows each utterance's hypotheses consumed into the oracle's restatements of
transducer_beam_boosted (decoding.py:428-495) and aed_beam_boosted
(decoding.py:502-587), keyed by the StepModel context (last token and frame
for the transducer, token prefix for AED).  n-best lists must agree exactly:
tokens, fp64 am / boost scores and traces.
"""

import numpy as np
import pytest

import gen_inputs as gi
from conftest import product_table, res_tuple

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def _cmp(got, exp):
    assert len(got) == len(exp)
    for g, e in zip(got, exp):
        g = res_tuple(g)
        assert g["tokens"] == e["tokens"]
        assert g["am"] == e["am"] and g["boost"] == e["boost"]
        assert g["trace"] == [list(x) for x in e["trace"]]


def _table(V, n, seed):
    phrases = gi.phrase_corpus(np.random.default_rng(seed), V, n)
    return product_table(phrases, V)


def _tbeam_case(lam, beam, cap, rollback=False, use_graph=False, B=5, T=9, V=48, seed=0, fused=True):
    import torch

    from paper_2508_07014_b200 import DecodeConfig
    from paper_2508_07014_b200.beams import StatelessTransducerModel, TransducerBeamDecoder

    tab = _table(V, 120, 1000 + seed)
    model = StatelessTransducerModel(V, enc_dim=32, pred_dim=32, joint_dim=32, seed=seed, blank_bias=0.5)
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    enc = torch.randn((B, T, 32), generator=g, device="cuda")
    lengths = np.random.default_rng(seed).integers(1, T + 1, size=B)
    cfg = DecodeConfig(lam=lam, beam_size=beam, max_symbols_per_frame=cap)
    dec = TransducerBeamDecoder(model, tab, cfg, B, T, use_graph=use_graph, rollback=rollback, fused=fused)
    assert dec.fused == fused
    out = dec.decode(model.project_encoder(enc), torch.from_numpy(lengths), record=True, want_trace=True)
    for b in range(B):
        rows = {}
        for lp, flags, last, t in out.records:
            if t[b] >= lengths[b]:
                continue
            for r in range(beam):
                if flags[b, r] & 1:
                    key = (int(last[b, r]), int(t[b]))
                    if key in rows:
                        assert np.array_equal(rows[key].view(np.uint32), lp[b, r].view(np.uint32))
                    rows[key] = lp[b, r].copy()

        def step(last, t):
            return rows[(-1 if last is None else int(last), t)]

        exp = orc.transducer_beam(step, int(lengths[b]), 0, tab, lam, beam, cap, V, rollback=rollback)
        _cmp(out.nbest[b], exp)
    return dec, out


@pytest.mark.parametrize("lam,beam,cap", [(1.0, 4, 2), (2.0, 3, 3), (0.0, 4, 2), (1.5, 8, 1), (1.0, 1, 2)])
@pytest.mark.parametrize("blobs", [0, 1])
def test_transducer_device_beam_matches_reference_by_replay(lam, beam, cap, blobs):
    """blobs = 0: closure data from the table's advance blobs (V <= 1024),
    1: closure records + bitmap marking (the path for larger vocabularies)."""
    from paper_2508_07014_b200 import _lib

    _lib.set_tuning("beam.blobs", blobs)
    try:
        _tbeam_case(lam, beam, cap)
    finally:
        _lib.set_tuning("beam.blobs", 0)


def test_transducer_device_beam_rollback():
    _tbeam_case(1.0, 4, 2, rollback=True, seed=3)


def test_transducer_device_beam_framework_joint():
    """The framework joint (torch gathers + log_softmax) instead of the fused
    beam-hidden and log-softmax kernels: same replay parity."""
    _tbeam_case(1.0, 4, 2, fused=False, seed=5)


def test_transducer_device_beam_graph_equals_eager():
    import torch

    from paper_2508_07014_b200 import DecodeConfig
    from paper_2508_07014_b200.beams import StatelessTransducerModel, TransducerBeamDecoder

    V, B, T = 64, 6, 11
    tab = _table(V, 200, 7)
    model = StatelessTransducerModel(V, enc_dim=32, pred_dim=32, joint_dim=32, seed=5, blank_bias=0.5)
    enc = model.project_encoder(torch.randn((B, T, 32), device="cuda", generator=torch.Generator("cuda").manual_seed(1)))
    lengths = torch.tensor([11, 3, 7, 11, 1, 9])
    cfg = DecodeConfig(lam=1.0, beam_size=4, max_symbols_per_frame=3)
    a = TransducerBeamDecoder(model, tab, cfg, B, T, use_graph=False).decode(enc, lengths, want_trace=True).nbest
    gd = TransducerBeamDecoder(model, tab, cfg, B, T, use_graph=True)
    b1 = gd.decode(enc, lengths, want_trace=True).nbest
    b2 = gd.decode(enc, lengths, want_trace=True).nbest  # graph replay after reset
    for x, y, z in zip(a, b1, b2):
        assert [res_tuple(r) for r in x] == [res_tuple(r) for r in y] == [res_tuple(r) for r in z]


def _aed_case(lam, beam, max_len, eos_bump=True, B=4, V=40, seed=0, rollback=False):
    import torch

    from paper_2508_07014_b200 import DecodeConfig
    from paper_2508_07014_b200.beams import AEDBeamDecoder, TransformerAEDModel, _walk

    tab = _table(V, 100, 2000 + seed)
    model = TransformerAEDModel(V, d_model=32, n_layers=2, n_heads=2, d_ff=64, max_len=max_len + 1, seed=seed)
    mem = torch.randn((B, 10, 32), device="cuda", generator=torch.Generator("cuda").manual_seed(seed))
    eos = V - 1
    cfg = DecodeConfig(lam=lam, beam_size=beam, eos_bump_enabled=eos_bump, rollback=rollback)
    dec = AEDBeamDecoder(model, tab, cfg, B, max_len=max_len, eos=eos, poll=1)
    out = dec.decode(mem, record=True, want_trace=True)
    for b in range(B):
        rows = {}
        for lp, hy, tr in out.records:
            for r in range(beam):
                f = int(hy["flags"][b, r])
                if (f & 1) and not (f & 2) and hy["len"][b, r] < max_len:
                    prefix = tuple(s[0] for s in _walk(tr, b, int(hy["node"][b, r])))
                    assert len(prefix) == hy["len"][b, r]
                    if prefix in rows:
                        assert np.array_equal(rows[prefix].view(np.uint32), lp[b, r].view(np.uint32))
                    rows[prefix] = lp[b, r].copy()
        exp = orc.aed_beam(lambda p, n: rows[tuple(p)], tab, lam, beam, max_len, eos, V, eos_bump=eos_bump,
                           rollback=rollback)
        _cmp(out.nbest[b], exp)


@pytest.mark.parametrize("lam,beam,max_len,bump", [(1.0, 4, 6, True), (2.0, 3, 5, True), (1.0, 4, 6, False),
                                                   (0.0, 4, 5, True), (1.0, 8, 4, True)])
def test_aed_device_beam_matches_reference_by_replay(lam, beam, max_len, bump):
    _aed_case(lam, beam, max_len, bump)


@pytest.mark.parametrize("bump", [True, False])
def test_aed_device_beam_rollback_extension(bump):
    """rollback=True (extension, parity unpinned): the eos step also takes
    back the state's backoff total; equal to the oracle's restatement."""
    _aed_case(1.0, 4, 6, bump, seed=4, rollback=True)


def test_device_beam_rejects_bad_config():
    import torch

    from paper_2508_07014_b200 import DecodeConfig
    from paper_2508_07014_b200.beams import StatelessTransducerModel, TransducerBeamDecoder

    tab = _table(32, 20, 3)
    model = StatelessTransducerModel(16, enc_dim=8, pred_dim=8, joint_dim=8)
    with pytest.raises(ValueError):
        TransducerBeamDecoder(model, tab, DecodeConfig(beam_size=4), 2, 4)
    model = StatelessTransducerModel(32, enc_dim=8, pred_dim=8, joint_dim=8)
    with pytest.raises(ValueError):
        TransducerBeamDecoder(model, tab, DecodeConfig(beam_size=33), 2, 4)
    del torch


def test_aed_device_beam_graphs_equal_eager():
    """AED decode steps captured as CUDA graphs (second run) and replayed
    (third run) give the eager run's n-best exactly."""
    import torch

    from paper_2508_07014_b200 import DecodeConfig
    from paper_2508_07014_b200.beams import AEDBeamDecoder, TransformerAEDModel

    V, B, max_len = 40, 4, 6
    tab = _table(V, 100, 2100)
    model = TransformerAEDModel(V, d_model=32, n_layers=2, n_heads=2, d_ff=64, max_len=max_len + 1, seed=2)
    mem = torch.randn((B, 10, 32), device="cuda", generator=torch.Generator("cuda").manual_seed(2))
    cfg = DecodeConfig(lam=1.0, beam_size=4)
    eager = AEDBeamDecoder(model, tab, cfg, B, max_len=max_len, eos=V - 1, use_graph=False).decode(
        mem, want_trace=True).nbest
    dec = AEDBeamDecoder(model, tab, cfg, B, max_len=max_len, eos=V - 1, use_graph=True)
    runs = [dec.decode(mem, want_trace=True).nbest for _ in range(3)]  # eager warm-up, capture, replay
    assert len(dec.graphs) > 0
    for r in runs:
        for x, y in zip(eager, r):
            assert [res_tuple(a) for a in x] == [res_tuple(a) for a in y]
