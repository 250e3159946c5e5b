"""Seeded synthetic inputs shared by the tests, the golden generator and bench.

Each generator replays the reference test-suite's RNG call sequence so the
same seed yields the same inputs as the reference's own fixtures:
  random_phrase_set / random_tree_spec  <- pkg/tests/conftest.py:43-65
  random_emissions                      <- pkg/tests/conftest.py:141-145
  phrase_corpus                         <- pkg/tests/test_acceptance.py:305-311
  random_transducer_rows                <- pkg/tests/test_decoding.py:101-108
  random_aed_rows                       <- pkg/tests/test_decoding.py:111-119
Golden fixtures store a sha256 of every generated input so a drift in the
generator (or in numpy's streams) fails loudly instead of silently.
"""

from __future__ import annotations

import hashlib

import numpy as np


def log_softmax(x) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    m = x.max(axis=-1, keepdims=True)
    return x - (m + np.log(np.exp(x - m).sum(axis=-1, keepdims=True)))


def random_phrase_set(rng, max_phrases=50, max_len=8, vocab_size=64):
    n = int(rng.integers(1, max_phrases + 1))
    out = set()
    for _ in range(n):
        length = int(rng.integers(1, max_len + 1))
        out.add(tuple(int(x) for x in rng.integers(0, vocab_size, size=length)))
    return sorted(out)


def random_tree_spec(rng, max_phrases=50, max_len=8, max_vocab=64, params=True):
    """(phrases, V, c0, beta) as conftest.random_tree draws them."""
    V = int(rng.integers(4, max_vocab + 1))
    ids = random_phrase_set(rng, max_phrases, max_len, V)
    if params:
        c0 = float(rng.uniform(0.1, 2.0))
        beta = float(rng.uniform(0.0, 3.0))
    else:
        c0, beta = 1.0, 2.0
    return ids, V, c0, beta


def random_emissions(rng, T, V, scale=2.0) -> np.ndarray:
    return log_softmax(rng.normal(0.0, scale, size=(T, V))).astype(np.float32)


def phrase_corpus(rng, V, count):
    """`count` distinct phrases of 1-3 words x 2-6 tokens in [1, V), sorted."""
    phrases = set()
    while len(phrases) < count:
        n_words = int(rng.integers(1, 4))
        length = sum(int(rng.integers(2, 7)) for _ in range(n_words))
        phrases.add(tuple(int(x) for x in rng.integers(1, V, size=length)))
    return sorted(phrases)


def random_transducer_rows(rng, V):
    """{context key: row} with keys '' and str(token), plus the default row."""
    rows = {str(ctx): log_softmax(rng.normal(0, 1.5, size=V)).astype(np.float32) for ctx in range(V)}
    rows[""] = log_softmax(rng.normal(0, 1.5, size=V)).astype(np.float32)
    default = log_softmax(rng.normal(0, 1.5, size=V)).astype(np.float32)
    return rows, default


def tied_rows(rng, n, V):
    """Rows with exact score ties across hypotheses: integer log-scores in
    {-4..-1} (the reference does not require normalised rows, and fp64 sums
    of small integers are exact, so different token sequences reach equal
    (combined, am) keys), every fourth row uniform (-2)."""
    z = -rng.integers(1, 5, size=(n, V)).astype(np.float32)
    z[::4] = -2.0
    return z


def tied_transducer_rows(rng, V):
    r = tied_rows(rng, V + 2, V)
    rows = {str(ctx): r[ctx] for ctx in range(V)}
    rows[""] = r[V]
    return rows, r[V + 1]


def tied_aed_rows(rng, V, n_rows=6):
    rows = {}
    r = tied_rows(rng, n_rows + 1, V)
    for i in range(n_rows):
        plen = int(rng.integers(0, 3))
        key = ",".join(str(int(x)) for x in rng.integers(0, V, size=plen))
        rows[key] = r[i]
    return rows, r[n_rows]


def random_aed_rows(rng, V, n_rows=6):
    rows = {}
    for _ in range(n_rows):
        plen = int(rng.integers(0, 3))
        key = ",".join(str(int(x)) for x in rng.integers(0, V, size=plen))
        rows[key] = log_softmax(rng.normal(0, 1.5, size=V)).astype(np.float32)
    default = log_softmax(rng.normal(0, 1.5, size=V)).astype(np.float32)
    return rows, default


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def phrases_sha(phrases) -> str:
    return hashlib.sha256(repr(list(map(tuple, phrases))).encode()).hexdigest()


# Standard corpora of the benchmark configs: fresh
# default_rng(1008) per corpus, TreeParams() defaults, unk = 0.
CORPORA = {
    "p100_v1024": (1024, 100),
    "p5k_v1024": (1024, 5000),
    "p20k_v1024": (1024, 20000),
    "p20k_v4096": (4096, 20000),
}


def corpus(name: str):
    V, n = CORPORA[name]
    return phrase_corpus(np.random.default_rng(1008), V, n), V


def reference_overhead_corpus():
    """The reference's decode-overhead corpus (test_acceptance.py:314-355),
    replaying its RNG call order exactly: default_rng(1008) -> the 20K and
    200-phrase corpora (:320, :326), two query-state draws of (100, 32)
    (:331-332, small table first), then 25 x (450 random targets, a seed)
    for synth_ctc_emissions(margin=0.5, boost_positions=[], blanks_between=3)
    (:342-353).  Returns (targets, seeds, S_small); the caller builds the
    emissions with its synth_ctc_emissions (acoustic.py:133-200 semantics)."""
    V = 1024
    rng = np.random.default_rng(1008)
    phrase_corpus(rng, V, 20_000)
    small = phrase_corpus(rng, V, 200)
    # the small table's state count: root + distinct prefixes (trie nodes)
    prefixes = {p[:i] for p in small for i in range(1, len(p) + 1)}
    s_small, s_big = 1 + len(prefixes), 140_870
    rng.integers(0, s_small, size=(100, 32))
    rng.integers(0, s_big, size=(100, 32))
    targets, seeds = [], []
    for _ in range(25):
        targets.append([int(x) for x in rng.integers(1, V, size=450)])
        seeds.append(int(rng.integers(2**31)))
    return targets, seeds, s_small
