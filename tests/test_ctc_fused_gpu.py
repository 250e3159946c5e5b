"""Fused speculative chunk-parallel greedy CTC (pgpb_ctc_spec.cu) vs the oracle.

The fused kernel decides every chunk of frames from a guessed start and
repairs the guesses in fix-up rounds; these tests drive the regimes that
stress that: phrase-dense emissions whose tree states stay deep across chunk
boundaries, heavy boosting that changes many decisions, long utterances that
run in several segments, every consumer-warp count, ragged lengths, small
trees whose root row is mostly unk (uncertified dense tokens -> warp rescans),
and vocabularies that are not a multiple of 4 (scalar row loads).  Results
must equal the reference restatement (oracle/pgpb_oracle.c, pinned to the
reference's compiled kernel) bit for bit: tokens, am, boost and the trace.
"""

import numpy as np
import pytest

import gen_inputs as gi
from conftest import product_table, res_tuple

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def _phrase_emissions(rng, phrases, T, V, noise=0.6, hit=4.0, blank_every=2):
    """Log-probs whose argmax path spells random phrases back to back (with
    blanks), plus near-miss competitors, so boosted states go deep."""
    logits = rng.normal(0.0, noise, size=(T, V))
    t = 0
    while t < T:
        ph = phrases[int(rng.integers(len(phrases)))]
        for tok in ph:
            if t >= T:
                break
            logits[t, tok] += hit
            logits[t, int(rng.integers(1, V))] += hit + float(rng.normal(0.0, 0.4))
            t += 1
            for _ in range(int(rng.integers(0, blank_every + 1))):
                if t >= T:
                    break
                logits[t, 0] += hit
                t += 1
    return gi.log_softmax(logits).astype(np.float32)


def _run(lps, lens, tab, lam, env=None):
    """Decode with the walker's code-path overrides (pgpb_set_tuning) set for
    this call only; the keys name the walker's modes."""
    from paper_2508_07014_b200 import DecodeConfig, _lib, ctc_greedy_boosted_batch

    for k, v in (env or {}).items():
        _lib.set_tuning(k, int(v))
    try:
        return ctc_greedy_boosted_batch(lps, lens, tab, DecodeConfig(lam=lam), blank_id=0, want_trace=True)
    finally:
        for k in (env or {}):
            _lib.set_tuning(k, 0)


def _check(got, lps, lens, tab, lam):
    for b in range(lps.shape[0]):
        n = lps.shape[1] if lens is None else int(lens[b])
        e = orc.ctc_greedy_decode(lps[b, :n], 0, tab, lam)
        g = res_tuple(got[b])
        assert g["tokens"] == e["tokens"], (b, lam)
        assert g["am"] == e["am"] and g["boost"] == e["boost"], (b, lam)
        assert g["trace"] == [list(x) for x in e["trace"]], (b, lam)


@pytest.fixture(scope="module")
def t20k():
    phrases, V = gi.corpus("p20k_v1024")
    return phrases, V, product_table(phrases, V)


@pytest.mark.parametrize("seq", ["0", "1", "2"])
@pytest.mark.parametrize("lam", [0.0, 1.0, 2.5])
def test_phrase_dense_deep_states(t20k, lam, seq):
    """seq: ctc.seq 0 = automatic mode choice, 1 = sequential walk,
    2 = speculative rounds only."""
    phrases, V, tab = t20k
    rng = np.random.default_rng(31)
    B, T = 24, 400
    lps = np.stack([_phrase_emissions(rng, phrases, T, V) for _ in range(B)])
    _check(_run(lps, None, tab, lam, {"ctc.seq": seq}), lps, None, tab, lam)


@pytest.mark.parametrize("env", [{"ctc.consumers": "1"}, {"ctc.consumers": "2"},
                                 {"ctc.consumers": "4"}, {"ctc.segment": "97"},
                                 {"ctc.segment": "300", "ctc.consumers": "3"},
                                 {"ctc.segment": "200", "ctc.seq": "1"},
                                 {"ctc.segment": "111", "ctc.seq": "2", "ctc.consumers": "1"}])
def test_segments_and_consumer_counts(t20k, env):
    phrases, V, tab = t20k
    rng = np.random.default_rng(32)
    B, T = 6, 1500
    lps = np.stack([_phrase_emissions(rng, phrases, T, V, blank_every=1) for _ in range(B)])
    lens = rng.integers(1, T + 1, size=B).astype(np.int32)
    lens[0] = T
    lens[1] = 1
    _check(_run(lps, lens, tab, 1.5, env), lps, lens, tab, 1.5)


@pytest.mark.parametrize("seq", ["0", "1", "2"])
@pytest.mark.parametrize("regime", ["dense", "blank3", "clean"])
def test_bench_regimes_vs_oracle(t20k, regime, seq):
    from paper_2508_07014_b200.acoustic import synth_ctc_emissions
    from paper_2508_07014_b200.context import Vocabulary

    phrases, V, tab = t20k
    rng = np.random.default_rng(33)
    B, T = 32, 200
    if regime == "clean":
        vocab = Vocabulary(tokens=tuple(str(i) for i in range(V)), blank_id=0)
        ems = []
        for _ in range(B):
            tgt = [int(x) for x in rng.integers(1, V, size=T // 4)]
            em = synth_ctc_emissions(tgt, vocab, margin=0.5, seed=int(rng.integers(2**31)), boost_positions=[],
                                     blanks_between=3)
            ems.append(em.logprobs[:T])
        T = min(e.shape[0] for e in ems)
        lps = np.stack([e[:T] for e in ems]).astype(np.float32)
    else:
        logits = rng.normal(0.0, 2.0, size=(B, T, V))
        if regime == "blank3":
            logits[:, np.arange(T) % 4 != 0, 0] += 10.0
        lps = gi.log_softmax(logits).astype(np.float32)
    for lam in (0.0, 1.0):
        _check(_run(lps, None, tab, lam, {"ctc.seq": seq}), lps, None, tab, lam)


def test_small_tree_unk_root_rows():
    """100-phrase tree: most tokens have no root arc (root score = unk), so
    the top-2 bound rarely certifies and the warp rescan path decides."""
    phrases, V = gi.corpus("p100_v1024")
    rng = np.random.default_rng(34)
    for unk in (0.0, -0.5, 0.7):
        tab = product_table(phrases, V, unk=unk)
        lps = np.stack([gi.random_emissions(rng, 150, V) for _ in range(8)])
        for lam in (0.7, 3.0):
            _check(_run(lps, None, tab, lam), lps, None, tab, lam)


@pytest.mark.parametrize("V", [1023, 37, 5])
def test_vocab_not_multiple_of_four(V):
    rng = np.random.default_rng(35 + V)
    phrases = gi.random_phrase_set(rng, 60 if V > 40 else 12, 6, V)
    tab = product_table(phrases, V)
    B, T = 10, 300
    lps = np.stack([_phrase_emissions(rng, phrases, T, V, noise=0.4) for _ in range(B)])
    lens = rng.integers(0, T + 1, size=B).astype(np.int32)
    for lam in (1.0, 4.0):
        _check(_run(lps, lens, tab, lam), lps, lens, tab, lam)


def test_empty_and_single_frame_batches(t20k):
    phrases, V, tab = t20k
    rng = np.random.default_rng(37)
    lps = np.stack([gi.random_emissions(rng, 5, V) for _ in range(7)])
    lens = np.array([0, 1, 0, 5, 2, 0, 1], dtype=np.int32)
    _check(_run(lps, lens, tab, 1.0), lps, lens, tab, 1.0)


def test_boost_sum_fallback_wide_dynamic_range(t20k):
    """Depth-1 arcs of 1e-7 and deeper arcs of ~1e6: the boost
    deltas span more than 53 bits, so the walker's exact tree sum must fall
    back to the sequential fp64 sum (still bit-exact)."""
    phrases, V, _ = t20k
    tab = product_table(phrases, V, c0=1e-7, beta=1e13)  # depth-1 arcs 1e-7, deeper arcs ~1e6
    rng = np.random.default_rng(38)
    B, T = 12, 300
    lps = np.stack([_phrase_emissions(rng, phrases, T, V) for _ in range(B)])
    got = _run(lps, None, tab, 1.0)
    _check(got, lps, None, tab, 1.0)
    assert any(abs(r.boost_score) > 1e5 for r in got)


@pytest.mark.parametrize("lam", [0.0, 1.0])
def test_am_sum_fallback_mixed_confidence(t20k, lam):
    """Near-certain frames (argmax log-prob ~ -1e-15) mixed with flat ones
    (~ -5): the log-probs span more than 53 bits, so the walker's exact tree
    sum of am must fall back to the sequential fp64 sum (bit-exact)."""
    phrases, V, tab = t20k
    rng = np.random.default_rng(39)
    B, T = 16, 250
    logits = rng.normal(0.0, 2.0, size=(B, T, V))
    peaky = rng.random((B, T)) < 0.3
    idx = rng.integers(0, V, size=(B, T))
    logits[peaky, idx[peaky]] += 45.0
    lps = gi.log_softmax(logits).astype(np.float32)
    lens = rng.integers(T // 2, T + 1, size=B).astype(np.int32)
    _check(_run(lps, lens, tab, lam), lps, lens, tab, lam)


@pytest.mark.parametrize("seq", ["0", "1"])
def test_vocab_4096_general_phase_a(seq):
    """V=4096 (the AED vocabulary): phase A's multi-tile path and the walker's
    48 KB shared root row, 20K-phrase tree."""
    phrases, V = gi.corpus("p20k_v4096")
    tab = product_table(phrases, V)
    rng = np.random.default_rng(40)
    B, T = 6, 160
    lps = np.stack([_phrase_emissions(rng, phrases, T, V) for _ in range(B)])
    lens = rng.integers(1, T + 1, size=B).astype(np.int32)
    for lam in (0.0, 1.0):
        _check(_run(lps, lens, tab, lam, {"ctc.seq": seq}), lps, lens, tab, lam)


@pytest.mark.parametrize("V", [1024, 64, 4])
def test_phase_a_ties_signed_zeros_masked(V):
    """Phase A's hardware warp reductions (redux.max.f32 over group maxima,
    then the first matching id) against the reference's first-max rules:
    quantised log-probs with exact ties for the argmax and the runner-up,
    duplicated maxima in different lanes / register groups, a maximum of
    -0.0 ahead of +0.0, and masked (-inf) tokens.  The signed-zero rows (two
    tokens of probability 1, not a distribution) are checked boosted too: the
    reference's float compares call -0.0 and +0.0 equal, so the lower id
    wins every tie the walker's warp keys see."""
    rng = np.random.default_rng(41 + V)
    if V == 1024:
        phrases, _ = gi.corpus("p20k_v1024")
    else:
        phrases = gi.random_phrase_set(rng, 12 if V > 8 else 3, 4, V)
    tab = product_table(phrases, V)
    B, T = 12, 180
    logits = np.round(rng.normal(0.0, 1.5, size=(B, T, V)) * 4.0) / 4.0
    lps = gi.log_softmax(logits).astype(np.float32)
    zeros = lps.copy()
    for b in range(B):
        for t in range(T):
            r = lps[b, t]
            kind = int(rng.integers(0, 6))
            if kind == 2 and V > 2:
                z = zeros[b, t]
                i, j = sorted(rng.choice(V, size=2, replace=False))
                z[:] = np.minimum(z, -1.0)
                z[i] = np.float32(-0.0)
                z[j] = np.float32(0.0)
                continue
            top = float(r.max())
            if kind == 1 and V > 2:  # duplicated maximum later in the row
                r[int(rng.integers(0, V))] = top
                r[int(rng.integers(0, V))] = top
            elif kind == 3:  # masked tokens (a finite maximum stays)
                m = rng.random(V) < 0.5
                m[int(np.argmax(r))] = False
                r[m] = -np.inf
            elif kind == 4 and V > 3:  # runner-up tie
                s = np.argsort(-r, kind="stable")
                r[int(rng.integers(0, V))] = r[s[1]]
    lens = rng.integers(1, T + 1, size=B).astype(np.int32)
    for lam in (0.0, 1.0, 2.5):
        _check(_run(lps, lens, tab, lam), lps, lens, tab, lam)
    for lam in (0.0, 1.0, 2.5):
        _check(_run(zeros, lens, tab, lam), zeros, lens, tab, lam)
