"""The oracle is pinned against the reference's own outputs (CPU only).

golden.json / golden.npz were produced by running the reference package
(tests/golden/gen_golden.py).  When oracle/_ref holds the reference's own
compiled Cython kernels, the C restatement is also compared with them on
fresh random inputs.
"""

import numpy as np
import pytest

import gen_inputs as gi
from conftest import golden, golden_npz, golden_tree_case, product_table

from oracle import oracle as orc

FIELDS = ["arc_from", "arc_token", "arc_to", "arc_weight", "state_start", "state_end", "backoff_to",
          "backoff_weight", "is_final", "final_score", "root_scores", "root_next"]


def bits_equal(a, b):
    a, b = np.asarray(a), np.asarray(b)
    if a.dtype.kind == "f":
        return a.shape == b.shape and np.array_equal(a.view(np.uint8), np.asarray(b, a.dtype).view(np.uint8))
    return np.array_equal(a, b)


@pytest.mark.parametrize("i", range(40))
def test_oracle_tables_and_advance_match_reference(i):
    g, phrases, V, c0, beta, unk, rng = golden_tree_case(i)
    z = golden_npz()
    t = orc.build_table(phrases, V, c0, beta, g["mode"], g["bonus"], unk)
    for f in FIELDS:
        assert bits_equal(getattr(t, f), z[f"tree{i}_{f}"]), f
    states = z[f"tree{i}_states"]
    sc, nx = orc.score_batch(t, states)
    assert bits_equal(sc, z[f"tree{i}_scores"])
    assert np.array_equal(nx, z[f"tree{i}_next"])


@pytest.mark.parametrize("name", ["p100_v1024", "p5k_v1024"])
def test_oracle_corpus_tables(name):
    g = golden()["corpora"][name]
    phrases, V = gi.corpus(name)
    assert gi.phrases_sha(phrases) == g["phrases_sha"]
    t = orc.build_table(phrases, V)
    assert t.num_states == g["S"]
    for f in FIELDS:
        assert gi.sha(np.asarray(getattr(t, f))) == g["arrays"][f], f
    states = np.random.default_rng(99).integers(0, t.num_states, size=512).astype(np.int32)
    sc, nx = orc.score_batch(t, states)
    assert gi.sha(sc) == g["advance_scores_sha"] and gi.sha(nx) == g["advance_next_sha"]


def _ctc_case(c):
    rng = np.random.default_rng(c["seed"])
    phrases, V, c0, beta = gi.random_tree_spec(rng, max_phrases=20, max_len=6, max_vocab=24)
    t = orc.build_table(phrases, V, c0, beta)
    T = int(rng.integers(3, 40))
    lp = gi.random_emissions(rng, T, V)
    assert gi.sha(lp) == c["lp_sha"]
    return t, lp


@pytest.mark.parametrize("j", range(40))
def test_oracle_ctc_greedy_matches_reference(j):
    c = golden()["ctc_greedy"][j]
    t, lp = _ctc_case(c)
    r = orc.ctc_greedy_decode(lp, 0, t, c["lam"])
    exp = c["result"]
    assert r["tokens"] == exp["tokens"] and r["am"] == exp["am"] and r["boost"] == exp["boost"]
    assert [list(x) for x in r["trace"]] == exp["trace"]
    r2 = orc.ctc_greedy_numpy(lp, 0, t, c["lam"])
    assert r2["tokens"] == exp["tokens"] and r2["am"] == exp["am"] and r2["boost"] == exp["boost"]


def test_oracle_config1_matches_reference():
    phrases, V = gi.corpus("p100_v1024")
    t = orc.build_table(phrases, V)
    rng = np.random.default_rng(0)
    lps = [gi.random_emissions(rng, 200, V) for _ in range(4)]
    for c in golden()["config1"]:
        lp = lps[c["utt"]]
        assert gi.sha(lp) == c["lp_sha"]
        r = orc.ctc_greedy_decode(lp, 0, t, c["lam"])
        assert r["tokens"] == c["result"]["tokens"] and r["am"] == c["result"]["am"]
        assert r["boost"] == c["result"]["boost"]


def _cmp_nbest(got, exp):
    assert len(got) == len(exp)
    for g, e in zip(got, exp):
        assert g["tokens"] == e["tokens"]
        assert g["am"] == e["am"] and g["boost"] == e["boost"]
        assert [list(x) for x in g["trace"]] == e["trace"]


@pytest.mark.parametrize("j", range(16))
def test_oracle_ctc_beam_matches_reference(j):
    c = golden()["ctc_beam"][j]
    rng = np.random.default_rng(c["seed"])
    phrases, V, c0, beta = gi.random_tree_spec(rng, max_phrases=12, max_len=5, max_vocab=16)
    t = orc.build_table(phrases, V, c0, beta)
    lp = gi.random_emissions(rng, int(rng.integers(3, 14)), V)
    assert gi.sha(lp) == c["lp_sha"]
    _cmp_nbest(orc.ctc_beam(lp, 0, t, c["lam"], c["beam"]), c["nbest"])


def transducer_case(c):
    rng = np.random.default_rng(c["seed"])
    phrases, V, c0, beta = gi.random_tree_spec(rng, max_phrases=10, max_len=4, max_vocab=12)
    t = orc.build_table(phrases, V, c0, beta)
    rows, default = gi.random_transducer_rows(rng, V)
    assert gi.sha(default, *[rows[k] for k in sorted(rows)]) == c["rows_sha"]

    def step(last, _t):
        return rows.get("" if last is None else str(int(last)), default)

    return t, step, V, phrases


@pytest.mark.parametrize("j", range(16))
def test_oracle_transducer_matches_reference(j):
    c = golden()["transducer_greedy"][j]
    t, step, V, _ = transducer_case(c)
    g = orc.transducer_greedy(step, c["T"], 0, t, c["lam"], c["cap"])
    e = c["result"]
    assert g["tokens"] == e["tokens"] and g["am"] == e["am"] and g["boost"] == e["boost"]
    assert [list(x) for x in g["trace"]] == e["trace"]
    cb = golden()["transducer_beam"][j]
    _cmp_nbest(orc.transducer_beam(step, c["T"], 0, t, c["lam"], cb["beam"], c["cap"], V), cb["nbest"])


def aed_case(c):
    rng = np.random.default_rng(c["seed"])
    phrases, V, c0, beta = gi.random_tree_spec(rng, max_phrases=10, max_len=4, max_vocab=12)
    t = orc.build_table(phrases, V, c0, beta)
    rows, default = gi.random_aed_rows(rng, V)
    assert gi.sha(default, *[rows[k] for k in sorted(rows)]) == c["rows_sha"]

    def step(prefix, _n):
        return rows.get(",".join(str(int(x)) for x in prefix), default)

    return t, step, V, phrases


@pytest.mark.parametrize("j", range(16))
def test_oracle_aed_beam_matches_reference(j):
    c = golden()["aed_beam"][j]
    t, step, V, _ = aed_case(c)
    _cmp_nbest(orc.aed_beam(step, t, c["lam"], c["beam"], c["max_len"], c["eos"], V, c["eos_bump"]), c["nbest"])


def test_oracle_matches_reference_cython_kernels():
    ref = orc.ref_kernels()
    if ref is None:
        pytest.skip("oracle/_ref not built (make -C oracle ref)")
    rng = np.random.default_rng(4242)
    for _ in range(20):
        phrases, V, c0, beta = gi.random_tree_spec(rng, max_phrases=40, max_len=8, max_vocab=64)
        t = orc.build_table(phrases, V, c0, beta, unk=float(rng.uniform(-0.5, 0.5)))
        st = rng.integers(0, t.num_states, size=33).astype(np.int32)
        a = orc.score_batch(t, st)
        b = ref.score_batch(*orc._tab_arrays(t), st)
        assert bits_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        lp = gi.random_emissions(rng, int(rng.integers(5, 60)), V)
        for lam in (0.0, 0.7, 2.0):
            x = orc.ctc_greedy(lp, 0, lam, lam != 0, t)
            y = ref.ctc_greedy(lp, 0, lam, lam != 0, *orc._tab_arrays(t))
            assert np.array_equal(x[0], y[0]) and x[1] == y[1] and x[2] == y[2]
            assert np.array_equal(x[3], y[3]) and np.array_equal(x[4], y[4])


def test_tdt_restatement_reduces_to_r7():
    """CPU-side sanity of the restatement: d = 0 on emissions, 1 on blanks == R7."""
    rng = np.random.default_rng(3)
    phrases, V, c0, beta = gi.random_tree_spec(rng, max_phrases=10, max_len=4, max_vocab=12)
    tab = product_table(phrases, V, c0, beta)
    rows, default = gi.random_transducer_rows(rng, V)

    def step(last, t):
        return rows.get("" if last is None else str(int(last)), default)

    def step_tdt(last, t):
        r = step(last, t)
        return r, (1 if int(np.argmax(r)) == 0 else 0)

    for lam in (0.0, 1.0):
        assert orc.transducer_greedy_tdt(step_tdt, 7, 0, tab, lam, 3) == orc.transducer_greedy(step, 7, 0, tab, lam, 3)
