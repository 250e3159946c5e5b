"""Beam decoders on the fused expansion + top-k kernel (GPU).

Golden vectors come from the reference's own beam decoders; the oracle's
restatements cover larger seeded cases.  On tie-free inputs tokens, traces
and scores are bit-identical (the fp64 candidate scores are computed with
the reference's operation order, the log-add-exp merges on the host).
"""

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
        assert g["am"] == e["am"] and g["boost"] == e["boost"]
        assert g["trace"] == [list(x) for x in e["trace"]]


@pytest.mark.parametrize("j", range(16))
def test_ctc_beam_matches_reference_golden(j):
    from paper_2508_07014_b200 import DecodeConfig, EmissionMatrix, ctc_beam_boosted

    c = golden()["ctc_beam"][j]
    rng = np.random.default_rng(c["seed"])
    phrases, V, c0, beta = gi.random_tree_spec(rng, max_phrases=12, max_len=5, max_vocab=16)
    tab = product_table(phrases, V, c0, beta)
    lp = gi.random_emissions(rng, int(rng.integers(3, 14)), V)
    best, nbest = ctc_beam_boosted(EmissionMatrix(lp, blank_id=0), tab,
                                   DecodeConfig(lam=c["lam"], beam_size=c["beam"]), want_trace=True)
    _cmp(nbest, c["nbest"])


@pytest.mark.parametrize("j", range(16))
def test_transducer_beam_matches_reference_golden(j):
    from paper_2508_07014_b200 import DecodeConfig, TableStepModel, transducer_beam_boosted

    c = golden()["transducer_beam"][j]
    rng = np.random.default_rng(c["seed"])
    phrases, V, c0, beta = gi.random_tree_spec(rng, max_phrases=10, max_len=4, max_vocab=12)
    tab = product_table(phrases, V, c0, beta)
    rows, default = gi.random_transducer_rows(rng, V)
    model = TableStepModel(flavor="transducer", default_row=default, rows=rows)
    best, nbest = transducer_beam_boosted(
        model, c["T"], 0, tab, DecodeConfig(lam=c["lam"], beam_size=c["beam"], max_symbols_per_frame=c["cap"]),
        want_trace=True)
    _cmp(nbest, c["nbest"])


@pytest.mark.parametrize("j", range(16))
def test_aed_beam_matches_reference_golden(j):
    from paper_2508_07014_b200 import DecodeConfig, TableStepModel, aed_beam_boosted

    c = golden()["aed_beam"][j]
    rng = np.random.default_rng(c["seed"])
    phrases, V, c0, beta = gi.random_tree_spec(rng, max_phrases=10, max_len=4, max_vocab=12)
    tab = product_table(phrases, V, c0, beta)
    rows, default = gi.random_aed_rows(rng, V)
    model = TableStepModel(flavor="aed", default_row=default, rows=rows, eos_id=c["eos"])
    best, nbest = aed_beam_boosted(model, tab, DecodeConfig(lam=c["lam"], beam_size=c["beam"],
                                                            eos_bump_enabled=c["eos_bump"]),
                                   max_len=c["max_len"], want_trace=True)
    _cmp(nbest, c["nbest"])


def test_ctc_beam_large_tree_vs_oracle():
    from paper_2508_07014_b200 import DecodeConfig, EmissionMatrix, ctc_beam_boosted

    phrases, V = gi.corpus("p5k_v1024")
    tab = product_table(phrases, V)
    small_v = 64
    rng = np.random.default_rng(31)
    # restrict to a V=64 slice of the corpus so the oracle's Python V-loop stays fast
    sub = [p for p in phrases if max(p) < small_v][:200] or [(1, 2, 3)]
    tab = product_table(sub, small_v)
    for beam in (4, 8, 16):
        lp = gi.random_emissions(rng, 20, small_v)
        best, nbest = ctc_beam_boosted(EmissionMatrix(lp, blank_id=0), tab, DecodeConfig(lam=1.0, beam_size=beam),
                                       want_trace=True)
        _cmp(nbest, orc.ctc_beam(lp, 0, tab, 1.0, beam))


def test_wide_beams_vs_oracle():
    from paper_2508_07014_b200 import DecodeConfig, EmissionMatrix, TableStepModel, aed_beam_boosted, \
        ctc_beam_boosted, transducer_beam_boosted

    rng = np.random.default_rng(41)
    phrases, V, c0, beta = gi.random_tree_spec(rng, max_phrases=10, max_len=4, max_vocab=8)
    tab = product_table(phrases, V, c0, beta)
    lp = gi.random_emissions(rng, 5, V)
    _, nb = ctc_beam_boosted(EmissionMatrix(lp, blank_id=0), tab, DecodeConfig(lam=1.0, beam_size=40), want_trace=True)
    _cmp(nb, orc.ctc_beam(lp, 0, tab, 1.0, 40))
    rows, default = gi.random_transducer_rows(rng, V)
    m = TableStepModel(flavor="transducer", default_row=default, rows=rows)
    step = lambda last, t: rows.get("" if last is None else str(int(last)), default)  # noqa: E731
    _, nb = transducer_beam_boosted(m, 3, 0, tab, DecodeConfig(lam=1.0, beam_size=40, max_symbols_per_frame=2),
                                    want_trace=True)
    _cmp(nb, orc.transducer_beam(step, 3, 0, tab, 1.0, 40, 2, V))
    arows, adef = gi.random_aed_rows(rng, V)
    am = TableStepModel(flavor="aed", default_row=adef, rows=arows, eos_id=V - 1)
    astep = lambda p, n: arows.get(",".join(map(str, p)), adef)  # noqa: E731
    _, nb = aed_beam_boosted(am, tab, DecodeConfig(lam=1.0, beam_size=40), max_len=3, want_trace=True)
    _cmp(nb, orc.aed_beam(astep, tab, 1.0, 40, 3, V - 1, V))


@pytest.mark.parametrize("beam", [64, 100])
def test_beam_64_and_wider_vs_oracle(beam):
    """Beam 64 (and 100: k = 200 candidates, 7 top-k passes) through the fused
    kernel on a 200-token vocabulary with a 300-phrase tree: n-best equal to
    the reference restatement (decoding.py:232-587)."""
    from paper_2508_07014_b200 import DecodeConfig, EmissionMatrix, TableStepModel, aed_beam_boosted, \
        ctc_beam_boosted, transducer_beam_boosted

    rng = np.random.default_rng(beam)
    V = 200
    tab = product_table(gi.phrase_corpus(rng, V, 300), V)
    lp = gi.random_emissions(rng, 10, V)
    _, nb = ctc_beam_boosted(EmissionMatrix(lp, blank_id=0), tab, DecodeConfig(lam=1.0, beam_size=beam),
                             want_trace=True)
    _cmp(nb, orc.ctc_beam(lp, 0, tab, 1.0, beam))
    rows, default = gi.random_transducer_rows(rng, V)
    m = TableStepModel(flavor="transducer", default_row=default, rows=rows)
    step = lambda last, t: rows.get("" if last is None else str(int(last)), default)  # noqa: E731
    _, nb = transducer_beam_boosted(m, 3, 0, tab, DecodeConfig(lam=1.0, beam_size=beam, max_symbols_per_frame=2),
                                    want_trace=True)
    _cmp(nb, orc.transducer_beam(step, 3, 0, tab, 1.0, beam, 2, V))
    arows, adef = gi.random_aed_rows(rng, V)
    am = TableStepModel(flavor="aed", default_row=adef, rows=arows, eos_id=V - 1)
    astep = lambda p, n: arows.get(",".join(map(str, p)), adef)  # noqa: E731
    _, nb = aed_beam_boosted(am, tab, DecodeConfig(lam=1.0, beam_size=beam), max_len=3, want_trace=True)
    _cmp(nb, orc.aed_beam(astep, tab, 1.0, beam, 3, V - 1, V))


def test_exhaustive_ctc_beam_lambda_zero():
    """Unpruned prefix beam equals exhaustive label-sequence search (reference test_06)."""
    import itertools
    import math

    from paper_2508_07014_b200 import DecodeConfig, EmissionMatrix, ctc_beam_boosted

    rng = np.random.default_rng(1006)
    for _ in range(3):
        T, V = int(rng.integers(3, 6)), int(rng.integers(3, 5))
        lp = gi.random_emissions(rng, T, V).astype(np.float64)
        totals = {}
        for path in itertools.product(range(V), repeat=T):
            out, prev = [], -1
            for s in path:
                if s != 0 and s != prev:
                    out.append(s)
                prev = s
            sc = sum(lp[t, s] for t, s in enumerate(path))
            k = tuple(out)
            o = totals.get(k)
            totals[k] = sc if o is None else max(o, sc) + math.log1p(math.exp(-abs(o - sc)))
        best_key = max(totals.items(), key=lambda kv: (kv[1], [-x for x in kv[0]]))[0]
        best, nbest = ctc_beam_boosted(EmissionMatrix(lp.astype(np.float32), blank_id=0), None,
                                       DecodeConfig(lam=0.0, beam_size=10**6))
        assert tuple(best.tokens) == best_key
        for r in nbest[:20]:
            assert r.am_score == pytest.approx(totals[tuple(r.tokens)], abs=1e-6)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_rollback_extension_reference_api_beams(seed):
    """DecodeConfig(rollback=True): an extension with no reference
    counterpart (parity unpinned), checked against the oracle's restatement:
    CTC / transducer beams add the state's backoff total to every hypothesis
    at the last frame, the AED beam to the eos step."""
    from paper_2508_07014_b200 import DecodeConfig, EmissionMatrix, TableStepModel, aed_beam_boosted, \
        ctc_beam_boosted, transducer_beam_boosted

    rng = np.random.default_rng(500 + seed)
    V = 48
    tab = product_table(gi.phrase_corpus(rng, V, 150), V)
    cfg = DecodeConfig(lam=1.0, beam_size=4, max_symbols_per_frame=2, rollback=True)
    lp = gi.random_emissions(rng, 12, V)
    _, nb = ctc_beam_boosted(EmissionMatrix(lp, blank_id=0), tab, cfg, want_trace=True)
    _cmp(nb, orc.ctc_beam(lp, 0, tab, 1.0, 4, rollback=True))
    rows, default = gi.random_transducer_rows(rng, V)
    m = TableStepModel(flavor="transducer", default_row=default, rows=rows)
    step = lambda last, t: rows.get("" if last is None else str(int(last)), default)  # noqa: E731
    _, nb = transducer_beam_boosted(m, 5, 0, tab, cfg, want_trace=True)
    _cmp(nb, orc.transducer_beam(step, 5, 0, tab, 1.0, 4, 2, V, rollback=True))
    arows, adef = gi.random_aed_rows(rng, V)
    am = TableStepModel(flavor="aed", default_row=adef, rows=arows, eos_id=V - 1)
    astep = lambda p, n: arows.get(",".join(map(str, p)), adef)  # noqa: E731
    _, nb = aed_beam_boosted(am, tab, cfg, max_len=4, want_trace=True)
    _cmp(nb, orc.aed_beam(astep, tab, 1.0, 4, 4, V - 1, V, rollback=True))
    # rollback actually changes something on this seed set
    _, plain = ctc_beam_boosted(EmissionMatrix(lp, blank_id=0), tab, DecodeConfig(lam=1.0, beam_size=4),
                                want_trace=True)
    assert [r.boost_score for r in plain] != [r.boost_score for r in ctc_beam_boosted(
        EmissionMatrix(lp, blank_id=0), tab, cfg)[1]] or seed != 0
