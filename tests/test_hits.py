"""Keyphrase hits (evaluation.py:90-134): the host restatement and the GPU
Aho-Corasick counter (pgpb_phrase_hits) against the reference's outputs on
seeded cases (tests/golden/hits_golden.json: overlapping, nested and
duplicate phrases, case folding, empty utterances and phrases), plus a
large random corpus where the GPU result must equal the host one."""

import json
from pathlib import Path

import numpy as np
import pytest

import hits_cases as hc

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "hits_golden.json").read_text())


def _rows(hits):
    return [[k, h.ref, h.hyp, h.tp, h.fp, h.fn] for k, h in hits.items()]


@pytest.mark.parametrize("seed", hc.SEEDS)
def test_host_hits_match_reference(seed):
    from paper_2508_07014_b200.evaluation import keyphrase_hits

    refs, hyps, phrases, ci = hc.case(seed)
    assert _rows(keyphrase_hits(refs, hyps, phrases, case_insensitive=ci)) == GOLD[str(seed)]


@pytest.mark.gpu
@pytest.mark.parametrize("seed", hc.SEEDS)
def test_device_hits_match_reference(seed):
    from paper_2508_07014_b200.evaluation import keyphrase_hits_device

    refs, hyps, phrases, ci = hc.case(seed)
    assert _rows(keyphrase_hits_device(refs, hyps, phrases, case_insensitive=ci)) == GOLD[str(seed)]


@pytest.mark.gpu
def test_device_hits_large_corpus_equals_host():
    from paper_2508_07014_b200.evaluation import keyphrase_hits, keyphrase_hits_device

    rng = np.random.default_rng(3)
    vocab = [f"w{i}" for i in range(60)]
    U = 3000
    refs = [[vocab[int(j)] for j in rng.integers(0, 60, size=int(rng.integers(0, 30)))] for _ in range(U)]
    hyps = [[vocab[int(j)] for j in rng.integers(0, 60, size=int(rng.integers(0, 30)))] for _ in range(U)]
    phrases = [" ".join(vocab[int(j)] for j in rng.integers(0, 60, size=int(rng.integers(1, 4)))) for _ in range(300)]
    assert _rows(keyphrase_hits_device(refs, hyps, phrases)) == _rows(keyphrase_hits(refs, hyps, phrases))
