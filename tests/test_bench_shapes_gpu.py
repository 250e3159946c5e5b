"""Replay parity at the benchmarked decoder shapes (BASELINE configs 2-4).

The decoders are built exactly as bench.py builds them (tests/
bench_workloads.py: same seeds, sizes, blank bias, eos offset, trees).  Every
log-prob row a hypothesis consumed is recorded on the device and replayed
into the oracle's restatements of the reference decoders, keyed by the
StepModel contract (acoustic.py:203-217: last token + frame for the
transducer, token prefix for AED):
  * config 2: LabelLoopingDecoder, 128 x 200 frames, 20K tree, LSTM-640,
    cap 5, every row -> transducer_greedy_boosted (decoding.py:350-393);
  * config 3: TransducerBeamDecoder, V=1024, 5K tree, beam 4, cap 5, batch
    64 (frames cut to 50 to bound the oracle's pure-Python V-loops), 8
    utterances -> transducer_beam_boosted (decoding.py:428-495);
  * config 4: AEDBeamDecoder, V=4096, 20K tree, beam 4, max_len 48, eos bump
    on, 4 utterances -> aed_beam_boosted (decoding.py:502-587).
Tokens, traces and fp64 scores must be identical.  The recording runs the
same kernels eagerly; the graph-replayed decode the bench times is checked
equal to it.
"""

import numpy as np
import pytest

import bench_workloads as bw
from conftest import res_tuple

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("lam", [1.0, 0.0])
def test_config2_label_looping_replay_at_bench_shape(lam):
    import torch

    from paper_2508_07014_b200 import DecodeConfig
    from paper_2508_07014_b200.rnnt import LabelLoopingDecoder
    from test_rnnt_gpu import _replay_check

    dev = torch.device("cuda", 0)
    model, tab, enc_proj = bw.config2(dev)
    c = bw.C2
    B, T = c["B"], c["T"]
    cfg = DecodeConfig(lam=lam)
    rec = LabelLoopingDecoder(model, tab, cfg, B, T, use_graph=False)
    o = rec.decode(enc_proj, record=True)
    assert int(o.num_out.sum()) > 10 * B  # the bench's emission rate, not an idle decode
    _replay_check(o, B, np.full(B, T), tab, lam, cfg.max_symbols_per_frame)
    # the graph-replayed decode the bench times gives the same outputs
    g = LabelLoopingDecoder(model, tab, cfg, B, T, use_graph=True)
    g.decode(enc_proj)
    og = g.decode(enc_proj)
    assert torch.equal(og.num_out, o.num_out) and torch.equal(og.am, o.am) and torch.equal(og.boost, o.boost)
    assert torch.equal(og.tokens, o.tokens) and torch.equal(og.states, o.states)
    if lam:
        assert float(o.boost.abs().max()) > 0.0


def _tbeam_replay(out, b, lengths, beam):
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
    return lambda last, t: rows[(-1 if last is None else int(last), t)]


def _cmp(got, exp):
    assert len(got) == len(exp)
    for g, e in zip(got, exp):
        g = res_tuple(g)
        assert g["tokens"] == e["tokens"]
        assert g["am"] == e["am"] and g["boost"] == e["boost"]
        assert g["trace"] == [list(x) for x in e["trace"]]


def test_config3_transducer_beam_replay_at_bench_shape():
    import torch

    from paper_2508_07014_b200 import DecodeConfig
    from paper_2508_07014_b200.beams import TransducerBeamDecoder

    dev = torch.device("cuda", 0)
    model, tab, enc = bw.config3(dev)
    c = bw.C3
    B, T_cut, V = c["B"], 50, tab.vocab_size
    cfg = DecodeConfig(lam=1.0, beam_size=c["beam"], max_symbols_per_frame=c["cap"])
    dec = TransducerBeamDecoder(model, tab, cfg, B, c["T"])
    lengths = np.full(B, T_cut)
    out = dec.decode(enc, torch.from_numpy(lengths), record=True, want_trace=True)
    for b in range(0, B, B // 8):
        step = _tbeam_replay(out, b, lengths, c["beam"])
        exp = orc.transducer_beam(step, T_cut, 0, tab, 1.0, c["beam"], c["cap"], V)
        _cmp(out.nbest[b], exp)
    # graph-replayed (bench) path equals the recorded run on the full batch
    g = TransducerBeamDecoder(model, tab, cfg, B, c["T"], use_graph=True)
    gb = g.decode(enc, torch.from_numpy(lengths), want_trace=True).nbest
    for x, y in zip(out.nbest, gb):
        assert [res_tuple(r) for r in x] == [res_tuple(r) for r in y]


def test_config4_aed_beam_replay_at_bench_shape():
    import torch

    from paper_2508_07014_b200 import DecodeConfig
    from paper_2508_07014_b200.beams import AEDBeamDecoder, _walk

    dev = torch.device("cuda", 0)
    model, tab, mem = bw.config4(dev)
    c = bw.C4
    B, max_len, beam, V = c["B"], c["max_len"], c["beam"], tab.vocab_size
    eos = V - 1
    cfg = DecodeConfig(lam=1.0, beam_size=beam)
    dec = AEDBeamDecoder(model, tab, cfg, B, max_len=max_len, eos=eos, poll=1, use_graph=False)
    out = dec.decode(mem, record=True, want_trace=True)
    lens = [len(nb[0].tokens) for nb in out.nbest]
    assert min(lens) < max_len  # hypotheses end on eos inside max_len
    for b in range(0, B, B // 4):
        rows = {}
        for lp, hy, tr in out.records:
            for r in range(beam):
                f = int(hy["flags"][b, r])
                if (f & 1) and not (f & 2) and hy["len"][b, r] < max_len:
                    prefix = tuple(s[0] for s in _walk(tr, b, int(hy["node"][b, r])))
                    if prefix in rows:
                        assert np.array_equal(rows[prefix].view(np.uint32), lp[b, r].view(np.uint32))
                    rows[prefix] = lp[b, r].copy()
        exp = orc.aed_beam(lambda p, n: rows[tuple(p)], tab, 1.0, beam, max_len, eos, V)
        _cmp(out.nbest[b], exp)
    # the graph-replayed decoder the bench times: same n-best
    g = AEDBeamDecoder(model, tab, cfg, B, max_len=max_len, eos=eos)
    runs = [g.decode(mem, want_trace=True).nbest for _ in range(3)]
    for r in runs:
        for x, y in zip(out.nbest, r):
            assert [res_tuple(a) for a in x] == [res_tuple(a) for a in y]
