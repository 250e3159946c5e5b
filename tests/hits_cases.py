"""Seeded keyphrase-hit cases (refs, hyps, phrases, case flag) shared by the
golden generator (tests/golden/gen_hits_golden.py, reference keyphrase_hits)
and tests/test_hits.py (ours, CPU and GPU)."""

import numpy as np

WORDS = ["the", "cat", "sat", "on", "mat", "a", "b", "New", "new", "york", "city", "is", "big", "x"]


def case(seed: int):
    rng = np.random.default_rng(seed)
    nw = int(rng.integers(3, len(WORDS) + 1))
    pool = WORDS[:nw]

    def sent():
        return [pool[int(i)] for i in rng.integers(0, nw, size=int(rng.integers(0, 25)))]

    U = int(rng.integers(1, 40))
    refs = [sent() for _ in range(U)]
    hyps = [sent() for _ in range(U)]
    phrases = []
    for _ in range(int(rng.integers(1, 15))):
        n = int(rng.integers(1, 4))
        phrases.append(" ".join(pool[int(i)] for i in rng.integers(0, nw, size=n)))
    phrases += ["a a", "a", "new york", "New York city", "  cat  sat ", ""]
    case_insensitive = bool(seed % 3 != 0)
    return refs, hyps, phrases, case_insensitive


SEEDS = list(range(30))
