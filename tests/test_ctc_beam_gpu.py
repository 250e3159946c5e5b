"""Batched device CTC prefix beam (pgpb_ctc_beam, beams.ctc_beam_batch) vs
the reference's ctc_beam_boosted (decoding.py:232-343).

Golden vectors from the reference itself and the oracle's restatement at
larger seeded sizes (20K / 5K trees, V=1024, ragged batches, beams 1-32).
Tokens, boosts, tree states and traces must be identical; am = logaddexp of
the prefix's blank / non-blank masses is accumulated with the device's
exp/log1p, so it is compared within 1e-12 relative (fp64, ulp-level; the
north_star bound for scores is 1e-5)."""

import numpy as np
import pytest

import gen_inputs as gi
from conftest import golden, product_table, res_tuple

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def _cmp(got, exp):
    assert len(got) == len(exp)
    for g, e in zip(got, exp):
        g = res_tuple(g)
        assert g["tokens"] == e["tokens"]
        assert g["boost"] == e["boost"]
        assert g["am"] == pytest.approx(e["am"], rel=1e-12, abs=1e-12)
        assert g["trace"] == [list(x) for x in e["trace"]]


def test_ctc_beam_batch_matches_reference_golden():
    from paper_2508_07014_b200 import DecodeConfig
    from paper_2508_07014_b200.beams import ctc_beam_batch

    for j in range(16):
        c = golden()["ctc_beam"][j]
        rng = np.random.default_rng(c["seed"])
        phrases, V, c0, beta = gi.random_tree_spec(rng, max_phrases=12, max_len=5, max_vocab=16)
        tab = product_table(phrases, V, c0, beta)
        lp = gi.random_emissions(rng, int(rng.integers(3, 14)), V)
        (best, nbest), = ctc_beam_batch(lp[None], None, tab, DecodeConfig(lam=c["lam"], beam_size=c["beam"]),
                                        blank_id=0, want_trace=True)
        _cmp(nbest, c["nbest"])


@pytest.mark.parametrize("beam", [1, 4, 8, 16, 32])
@pytest.mark.parametrize("corpus", ["p5k_v1024", "p20k_v1024"])
def test_ctc_beam_batch_vs_oracle(corpus, beam):
    from paper_2508_07014_b200 import DecodeConfig
    from paper_2508_07014_b200.beams import ctc_beam_batch

    phrases, V = gi.corpus(corpus)
    tab = product_table(phrases, V)
    rng = np.random.default_rng(beam)
    B, T = 5, 30 if beam <= 8 else 14
    lps = np.stack([gi.random_emissions(rng, T, V) for _ in range(B)])
    lens = np.array([T, 1, 0, T - 3, T // 2], np.int32)
    for lam in (1.0, 0.0):
        out = ctc_beam_batch(lps, lens, tab, DecodeConfig(lam=lam, beam_size=beam), blank_id=0, want_trace=True)
        for b in range(B):
            exp = orc.ctc_beam(lps[b, :lens[b]], 0, tab, lam, beam)
            _cmp(out[b][1], exp)


def test_ctc_beam_batch_phrase_emissions_deep_states():
    """Emissions that spell tree phrases: prefixes run deep into the tree and
    boosting reorders the beam."""
    from test_ctc_fused_gpu import _phrase_emissions

    from paper_2508_07014_b200 import DecodeConfig
    from paper_2508_07014_b200.beams import ctc_beam_batch

    phrases, V = gi.corpus("p20k_v1024")
    tab = product_table(phrases, V)
    rng = np.random.default_rng(9)
    B, T = 4, 24
    lps = np.stack([_phrase_emissions(rng, phrases, T, V, noise=0.8, hit=2.0) for _ in range(B)])
    out = ctc_beam_batch(lps, None, tab, DecodeConfig(lam=1.5, beam_size=8), blank_id=0, want_trace=True)
    for b in range(B):
        _cmp(out[b][1], orc.ctc_beam(lps[b], 0, tab, 1.5, 8))
    assert any(s.state != 0 and s.boost > 1.5 for r in out for s in (r[0].trace or []))  # deep arcs taken


def test_ctc_beam_batch_no_table_and_errors():
    import torch

    from paper_2508_07014_b200 import DecodeConfig
    from paper_2508_07014_b200.beams import ctc_beam_batch

    rng = np.random.default_rng(3)
    lps = np.stack([gi.random_emissions(rng, 9, 12) for _ in range(3)])
    out = ctc_beam_batch(lps, None, None, DecodeConfig(beam_size=4), blank_id=0, want_trace=True)
    for b in range(3):
        _cmp(out[b][1], orc.ctc_beam(lps[b], 0, None, 1.0, 4))
    with pytest.raises(ValueError):
        ctc_beam_batch(lps, [9, 10, 1], None, DecodeConfig(beam_size=4), blank_id=0)
    with pytest.raises(ValueError):
        ctc_beam_batch(torch.zeros((2, 3, 12)), None, None, DecodeConfig(beam_size=33), blank_id=0)


def test_ctc_beam_batch_rollback_extension():
    """rollback=True (extension, parity unpinned): equal to the oracle's
    restatement (backoff total added to every prefix after the last frame)."""
    from paper_2508_07014_b200 import DecodeConfig
    from paper_2508_07014_b200.beams import ctc_beam_batch

    phrases, V = gi.corpus("p5k_v1024")
    tab = product_table(phrases, V)
    rng = np.random.default_rng(44)
    lps = np.stack([gi.random_emissions(rng, 20, V) for _ in range(4)])
    out = ctc_beam_batch(lps, None, tab, DecodeConfig(lam=1.0, beam_size=4, rollback=True), blank_id=0,
                         want_trace=True)
    for b in range(4):
        _cmp(out[b][1], orc.ctc_beam(lps[b], 0, tab, 1.0, 4, rollback=True))


@pytest.mark.parametrize("beam", [4, 8])
def test_ctc_beam_batch_masked_rows(beam):
    """Rows with most tokens at -inf (fewer finite candidates per warp than
    the beam, so the fp32 prefilter's warp bound is -inf) and a few frames
    where only blank is finite; boosted and unboosted vs the oracle."""
    from paper_2508_07014_b200 import DecodeConfig
    from paper_2508_07014_b200.beams import ctc_beam_batch

    phrases, V = gi.corpus("p20k_v1024")
    tab = product_table(phrases, V)
    rng = np.random.default_rng(70 + beam)
    B, T = 4, 16
    lps = np.stack([gi.random_emissions(rng, T, V) for _ in range(B)])
    for b in range(B):
        for t in range(T):
            keep = rng.choice(V, size=int(rng.integers(1, 9)), replace=False)
            row = np.full(V, -np.inf, np.float32)
            row[keep] = lps[b, t, keep]
            row[0] = lps[b, t, 0]
            if t % 5 == 4:
                row[1:] = -np.inf
            lps[b, t] = row
    lens = np.array([T, T - 1, 2, 1], np.int32)
    for lam in (1.0, 0.0):
        out = ctc_beam_batch(lps, lens, tab, DecodeConfig(lam=lam, beam_size=beam), blank_id=0, want_trace=True)
        for b in range(B):
            _cmp(out[b][1], orc.ctc_beam(lps[b, :lens[b]], 0, tab, lam, beam))
