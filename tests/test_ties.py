"""Beam decoders on inputs with exact score ties, against the reference.

tests/golden/ties_golden.json holds the reference's own n-best lists
(gen_ties_golden.py) for integer-valued rows (exact fp64 sums): many candidates
of different hypotheses share (combined score, am), and the reference's
token-tuple order (decoding.py:323-327, :407-411) decides which survive.
The oracle is pinned on them (CPU), and the drop-in beams are checked
bit-exact (GPU): their device top-k extends its cut by the whole tie group
and the host re-ranks with the full key.
"""

import json
from functools import lru_cache
from pathlib import Path

import numpy as np
import pytest

import gen_inputs as gi
from conftest import product_table, res_tuple

from oracle import oracle as orc

HERE = Path(__file__).resolve().parent


@lru_cache(maxsize=1)
def ties():
    return json.loads((HERE / "golden" / "ties_golden.json").read_text())


def _cmp(got, exp):
    assert len(got) == len(exp)
    for g, e in zip(got, exp):
        assert g["tokens"] == e["tokens"]
        assert g["am"] == e["am"] and g["boost"] == e["boost"]
        assert [list(x) for x in g["trace"]] == e["trace"]


def ctc_case(c, build):
    rng = np.random.default_rng(c["seed"])
    phrases, V, c0, beta = gi.random_tree_spec(rng, max_phrases=12, max_len=5, max_vocab=16)
    tab = build(phrases, V, c0, beta)
    lp = gi.tied_rows(rng, int(rng.integers(3, 12)), V)
    assert gi.sha(lp) == c["lp_sha"], "input generator drifted"
    return tab, lp, V


def transducer_case(c, build):
    rng = np.random.default_rng(c["seed"])
    phrases, V, c0, beta = gi.random_tree_spec(rng, max_phrases=10, max_len=4, max_vocab=12)
    tab = build(phrases, V, c0, beta)
    rows, default = gi.tied_transducer_rows(rng, V)
    assert gi.sha(default, *[rows[k] for k in sorted(rows)]) == c["rows_sha"], "input generator drifted"
    return tab, rows, default, V


def aed_case(c, build):
    rng = np.random.default_rng(c["seed"])
    phrases, V, c0, beta = gi.random_tree_spec(rng, max_phrases=10, max_len=4, max_vocab=12)
    V = max(V, 4)
    tab = build(phrases, V, c0, beta)
    rows, default = gi.tied_aed_rows(rng, V)
    assert gi.sha(default, *[rows[k] for k in sorted(rows)]) == c["rows_sha"], "input generator drifted"
    return tab, rows, default, V


def test_inputs_really_tie():
    """Each case family has candidates of different hypotheses with equal
    (combined, am): the tie-break is exercised, not vacuous."""
    lp = gi.tied_rows(np.random.default_rng(0), 8, 12)
    assert all(len(set(r.tolist())) <= 4 for r in lp)
    assert float(lp[1][0]) + float(lp[2][1]) in {float(a) + float(b) for a in lp[1][1:] for b in lp[2]}


@pytest.mark.parametrize("j", range(12))
def test_oracle_ctc_beam_ties(j):
    c = ties()["ctc_beam"][j]
    t, lp, _ = ctc_case(c, orc.build_table)
    _cmp(orc.ctc_beam(lp, 0, t, c["lam"], c["beam"]), c["nbest"])


@pytest.mark.parametrize("j", range(12))
def test_oracle_transducer_beam_ties(j):
    c = ties()["transducer_beam"][j]
    t, rows, default, V = transducer_case(c, orc.build_table)

    def step(last, _t):
        return rows.get("" if last is None else str(int(last)), default)

    _cmp(orc.transducer_beam(step, c["T"], 0, t, c["lam"], c["beam"], c["cap"], V), c["nbest"])


@pytest.mark.parametrize("j", range(12))
def test_oracle_aed_beam_ties(j):
    c = ties()["aed_beam"][j]
    t, rows, default, V = aed_case(c, orc.build_table)

    def step(prefix, _n):
        return rows.get(",".join(str(int(x)) for x in prefix), default)

    _cmp(orc.aed_beam(step, t, c["lam"], c["beam"], c["max_len"], c["eos"], V, c["eos_bump"]), c["nbest"])


@pytest.mark.gpu
@pytest.mark.parametrize("j", range(12))
def test_ctc_beam_ties(j):
    from paper_2508_07014_b200 import DecodeConfig, EmissionMatrix, ctc_beam_boosted

    c = ties()["ctc_beam"][j]
    tab, lp, _ = ctc_case(c, product_table)
    _, nbest = ctc_beam_boosted(EmissionMatrix(lp, blank_id=0), tab, DecodeConfig(lam=c["lam"], beam_size=c["beam"]),
                                want_trace=True)
    _cmp([res_tuple(r) for r in nbest], c["nbest"])


@pytest.mark.gpu
@pytest.mark.parametrize("j", range(12))
def test_transducer_beam_ties(j):
    from paper_2508_07014_b200 import DecodeConfig, TableStepModel, transducer_beam_boosted

    c = ties()["transducer_beam"][j]
    tab, rows, default, _ = transducer_case(c, product_table)
    model = TableStepModel(flavor="transducer", default_row=default, rows=rows)
    _, nbest = transducer_beam_boosted(model, c["T"], 0, tab, DecodeConfig(lam=c["lam"], beam_size=c["beam"],
                                                                           max_symbols_per_frame=c["cap"]),
                                       want_trace=True)
    _cmp([res_tuple(r) for r in nbest], c["nbest"])


@pytest.mark.gpu
@pytest.mark.parametrize("j", range(12))
def test_aed_beam_ties(j):
    from paper_2508_07014_b200 import DecodeConfig, TableStepModel, aed_beam_boosted

    c = ties()["aed_beam"][j]
    tab, rows, default, _ = aed_case(c, product_table)
    model = TableStepModel(flavor="aed", default_row=default, rows=rows, eos_id=c["eos"])
    _, nbest = aed_beam_boosted(model, tab, DecodeConfig(lam=c["lam"], beam_size=c["beam"],
                                                         eos_bump_enabled=c["eos_bump"]),
                                max_len=c["max_len"], want_trace=True)
    _cmp([res_tuple(r) for r in nbest], c["nbest"])
