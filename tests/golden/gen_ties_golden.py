"""Golden vectors for the beam decoders on inputs with exact score ties,
made by running the REFERENCE (same setup as gen_golden.py):

    python tests/golden/gen_ties_golden.py [--ref-src /tmp/refpkg/src]

Rows are integer log-scores (tests/gen_inputs.py::tied_rows), so
many candidates of different hypotheses share (combined score, am) and the
reference's token-tuple order decides which survive (decoding.py:323-327,
:407-411).  Output: tests/golden/ties_golden.json.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE))
import gen_inputs as gi  # noqa: E402
from gen_golden import ensure_ref  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref-src", type=Path, default=None)
    args = ap.parse_args()
    sys.path.insert(0, str(ensure_ref(args.ref_src)))
    from phraseboost.acoustic import EmissionMatrix, TableStepModel
    from phraseboost.context import ContextList, Phrase
    from phraseboost.decoding import DecodeConfig, aed_beam_boosted, ctc_beam_boosted, transducer_beam_boosted
    from phraseboost.table import compile_arc_table
    from phraseboost.tree import TreeParams, build_prefix_tree, compute_fail_links

    def table_of(phrases, V, c0, beta):
        ctx = ContextList(phrases=[Phrase(" ".join(map(str, p)), tuple(p)) for p in phrases], min_chars=0)
        return compile_arc_table(compute_fail_links(build_prefix_tree(ctx, TreeParams(c0=c0, beta=beta), V)))

    def res_dict(res):
        return {"tokens": [int(x) for x in res.tokens], "am": float(res.am_score), "boost": float(res.boost_score),
                "trace": [[int(s.token), float(s.boost), int(s.state)] for s in (res.trace or [])]}

    meta = {"note": "beam decoders of the reference on tie-heavy rows (gen_ties_golden.py)"}
    cases = []
    for i in range(12):
        seed = 9600 + i
        rng = np.random.default_rng(seed)
        phrases, V, c0, beta = gi.random_tree_spec(rng, max_phrases=12, max_len=5, max_vocab=16)
        tab = table_of(phrases, V, c0, beta)
        T = int(rng.integers(3, 12))
        lp = gi.tied_rows(rng, T, V)
        lam = float(rng.choice([0.0, 1.0]))
        beam = int(rng.choice([2, 3, 4, 8]))
        best, nbest = ctc_beam_boosted(EmissionMatrix(lp, blank_id=0), tab, DecodeConfig(lam=lam, beam_size=beam),
                                       want_trace=True)
        cases.append({"seed": seed, "T": T, "lam": lam, "beam": beam, "lp_sha": gi.sha(lp),
                      "nbest": [res_dict(r) for r in nbest]})
    meta["ctc_beam"] = cases
    cases = []
    for i in range(12):
        seed = 9700 + i
        rng = np.random.default_rng(seed)
        phrases, V, c0, beta = gi.random_tree_spec(rng, max_phrases=10, max_len=4, max_vocab=12)
        tab = table_of(phrases, V, c0, beta)
        rows, default = gi.tied_transducer_rows(rng, V)
        model = TableStepModel(flavor="transducer", default_row=default, rows=rows)
        T = int(rng.integers(2, 6))
        cap = int(rng.integers(1, 4))
        lam = float(rng.choice([0.0, 1.0]))
        beam = int(rng.choice([2, 3, 4]))
        best, nbest = transducer_beam_boosted(model, T, 0, tab,
                                              DecodeConfig(lam=lam, beam_size=beam, max_symbols_per_frame=cap),
                                              want_trace=True)
        cases.append({"seed": seed, "T": T, "cap": cap, "lam": lam, "beam": beam,
                      "rows_sha": gi.sha(default, *[rows[k] for k in sorted(rows)]),
                      "nbest": [res_dict(r) for r in nbest]})
    meta["transducer_beam"] = cases
    cases = []
    for i in range(12):
        seed = 9800 + i
        rng = np.random.default_rng(seed)
        phrases, V, c0, beta = gi.random_tree_spec(rng, max_phrases=10, max_len=4, max_vocab=12)
        V = max(V, 4)
        tab = table_of(phrases, V, c0, beta)
        rows, default = gi.tied_aed_rows(rng, V)
        eos = V - 1
        model = TableStepModel(flavor="aed", default_row=default, rows=rows, eos_id=eos)
        max_len = int(rng.integers(2, 5))
        lam = float(rng.choice([0.0, 1.0]))
        beam = int(rng.choice([2, 3, 4]))
        bump = bool(i % 3 != 2)
        best, nbest = aed_beam_boosted(model, tab, DecodeConfig(lam=lam, beam_size=beam, eos_bump_enabled=bump),
                                       max_len=max_len, want_trace=True)
        cases.append({"seed": seed, "eos": eos, "max_len": max_len, "lam": lam, "beam": beam, "eos_bump": bump,
                      "rows_sha": gi.sha(default, *[rows[k] for k in sorted(rows)]),
                      "nbest": [res_dict(r) for r in nbest]})
    meta["aed_beam"] = cases
    (HERE / "ties_golden.json").write_text(json.dumps(meta, indent=1, sort_keys=True))
    print("wrote", HERE / "ties_golden.json")


if __name__ == "__main__":
    main()
