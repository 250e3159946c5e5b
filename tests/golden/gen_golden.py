"""Generate the golden vectors by running the REFERENCE implementation.

Run in the build container (needs /root/reference):

    python tests/golden/gen_golden.py [--ref-src /tmp/refpkg/src]

It copies /root/reference/pkg to a scratch dir (the reference tree is
read-only), builds its Cython extension there (pkg/setup.py), imports the
`phraseboost` package from that copy and records, for seeded inputs from
tests/gen_inputs.py:
  * compiled tables (all ArcTable arrays) of random trees and of the four
    benchmark corpora (arrays for small trees, sha256 for large ones);
  * get_scores_batch outputs (sha256 + a few explicit cells);
  * decoder outputs of ctc_greedy_boosted (compiled and NumPy backends),
    ctc_beam_boosted, transducer_greedy_boosted, transducer_beam_boosted and
    aed_beam_boosted, with traces;
  * synth_ctc_emissions outputs (sha256).
Outputs: tests/golden/golden.json and tests/golden/golden.npz.  Nothing
under /root/reference is copied into the repository; only outputs.
"""

from __future__ import annotations

import argparse
import json
import shutil
import subprocess
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
import gen_inputs as gi  # noqa: E402


def ensure_ref(src: Path | None) -> Path:
    if src is not None and (src / "phraseboost").exists():
        return src
    dst = Path("/tmp/pgpb_golden_ref")
    if not (dst / "src" / "phraseboost").exists():
        shutil.rmtree(dst, ignore_errors=True)
        shutil.copytree("/root/reference/pkg", dst)
        subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=dst, check=True,
                       capture_output=True)
    return dst / "src"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref-src", type=Path, default=None)
    args = ap.parse_args()
    sys.path.insert(0, str(ensure_ref(args.ref_src)))
    import phraseboost as pb
    from phraseboost import _backend
    from phraseboost.acoustic import EmissionMatrix, TableStepModel, synth_ctc_emissions
    from phraseboost.context import ContextList, Phrase, Vocabulary
    from phraseboost.decoding import (DecodeConfig, aed_beam_boosted, ctc_beam_boosted,
                                      ctc_greedy_boosted, transducer_beam_boosted,
                                      transducer_greedy_boosted)
    from phraseboost.table import compile_arc_table, get_scores_batch
    from phraseboost.tree import TreeParams, build_prefix_tree, compute_fail_links

    assert _backend.backend_name() == "compiled", "reference Cython extension not built"
    npz: dict[str, np.ndarray] = {}
    meta: dict = {"reference": "phraseboost " + pb.__version__, "numpy": np.__version__}
    FIELDS = ["arc_from", "arc_token", "arc_to", "arc_weight", "state_start", "state_end",
              "backoff_to", "backoff_weight", "is_final", "final_score", "root_scores", "root_next"]

    def table_of(phrases, V, c0=1.0, beta=2.0, mode="depth_scaled", bonus=0.0, unk=0.0):
        ctx = ContextList(phrases=[Phrase(" ".join(map(str, p)), tuple(p)) for p in phrases], min_chars=0)
        params = TreeParams(c0=c0, beta=beta, weight_mode=mode, uniform_final_bonus=bonus)
        tree = compute_fail_links(build_prefix_tree(ctx, params, V))
        return tree, compile_arc_table(tree, unk_score=unk)

    def trace_list(res):
        return [[int(s.token), float(s.boost), int(s.state)] for s in (res.trace or [])]

    def res_dict(res):
        return {"tokens": [int(x) for x in res.tokens], "am": float(res.am_score),
                "boost": float(res.boost_score), "trace": trace_list(res)}

    # --- random trees: full arrays + advance -------------------------------------
    trees = []
    for i in range(40):
        seed = 7000 + i
        rng = np.random.default_rng(seed)
        mode = "uniform" if i % 8 == 7 else "depth_scaled"
        phrases, V, c0, beta = gi.random_tree_spec(rng, max_phrases=50, max_len=8, max_vocab=64)
        unk = float(rng.choice([0.0, 0.3, -0.2]))
        bonus = 0.0
        tree, tab = table_of(phrases, V, c0, beta, mode, bonus, unk)
        states = rng.integers(0, tab.num_states, size=24).astype(np.int32)
        res = get_scores_batch(tab, states)
        for f in FIELDS:
            npz[f"tree{i}_{f}"] = np.asarray(getattr(tab, f))
        npz[f"tree{i}_states"] = states
        npz[f"tree{i}_scores"] = res.scores
        npz[f"tree{i}_next"] = res.next_states
        npz[f"tree{i}_acc"] = np.array([n.acc_score for n in tree.nodes])
        trees.append({"seed": seed, "V": V, "c0": c0, "beta": beta, "mode": mode, "bonus": bonus,
                      "unk": unk, "phrases_sha": gi.phrases_sha(phrases), "S": tab.num_states,
                      "dump": tree.dump() if i < 3 else None})
    meta["trees"] = trees

    # --- benchmark corpora: hashes ----------------------------------------------
    corp = {}
    for name in gi.CORPORA:
        phrases, V = gi.corpus(name)
        tree, tab = table_of(phrases, V)
        rng = np.random.default_rng(99)
        states = rng.integers(0, tab.num_states, size=512).astype(np.int32)
        res = get_scores_batch(tab, states)
        corp[name] = {
            "V": V, "phrases_sha": gi.phrases_sha(phrases), "S": tab.num_states, "A": tab.num_arcs,
            "max_depth": tree.max_depth,
            "arrays": {f: gi.sha(np.asarray(getattr(tab, f))) for f in FIELDS},
            "advance_states_sha": gi.sha(states),
            "advance_scores_sha": gi.sha(res.scores), "advance_next_sha": gi.sha(res.next_states),
            "cells": [[int(b), int(v), float(res.scores[b, v]), int(res.next_states[b, v])]
                      for b, v in zip(rng.integers(0, 512, 64), rng.integers(0, V, 64))],
        }
    meta["corpora"] = corp

    # --- greedy CTC ---------------------------------------------------------------
    ctc = []
    for i in range(40):
        seed = 8000 + i
        rng = np.random.default_rng(seed)
        phrases, V, c0, beta = gi.random_tree_spec(rng, max_phrases=20, max_len=6, max_vocab=24)
        _, tab = table_of(phrases, V, c0, beta)
        T = int(rng.integers(3, 40))
        lp = gi.random_emissions(rng, T, V)
        lam = float(rng.choice([0.0, 0.3, 1.0, 2.0]))
        em = EmissionMatrix(logprobs=lp, blank_id=0)
        r_c = ctc_greedy_boosted(em, tab, DecodeConfig(lam=lam), want_trace=True)
        with _backend.forced_backend("python"):
            r_p = ctc_greedy_boosted(em, tab, DecodeConfig(lam=lam), want_trace=True)
        assert res_dict(r_c) == res_dict(r_p)
        ctc.append({"seed": seed, "V": V, "c0": c0, "beta": beta, "T": T, "lam": lam,
                    "lp_sha": gi.sha(lp), "result": res_dict(r_c)})
    meta["ctc_greedy"] = ctc

    # config 1: 100-phrase tree, V=1024, 4 x 200 frames, default_rng(0)
    phrases, V = gi.corpus("p100_v1024")
    _, tab = table_of(phrases, V)
    rng = np.random.default_rng(0)
    c1 = []
    lps = [gi.random_emissions(rng, 200, V) for _ in range(4)]
    for lam in (0.0, 1.0):
        for u, lp in enumerate(lps):
            r = ctc_greedy_boosted(EmissionMatrix(lp, blank_id=0), tab, DecodeConfig(lam=lam), want_trace=True)
            c1.append({"utt": u, "lam": lam, "lp_sha": gi.sha(lp), "result": res_dict(r)})
    meta["config1"] = c1

    # --- synth emissions ------------------------------------------------------------
    letters = "abcdefghijklmnopqrstuvwxyz"
    vocab = Vocabulary(tokens=("<b>",) + tuple(letters) + (" ",), blank_id=0)
    syn = []
    for j, (word, margin, bp, blanks) in enumerate([("cat", 0.5, None, 1), ("dog", 1.5, [0, 1], 2),
                                                     ("lemur", 0.5, [], 3)]):
        tgt = [vocab.id_of(c) for c in word]
        em = synth_ctc_emissions(tgt, vocab, margin=margin, seed=40 + j, boost_positions=bp,
                                 distractor_pool=[vocab.id_of(c) for c in "qxz"], blanks_between=blanks)
        syn.append({"word": word, "margin": margin, "boost_positions": bp, "blanks": blanks,
                    "seed": 40 + j, "sha": gi.sha(em.logprobs)})
    meta["synth"] = syn

    # --- beams ----------------------------------------------------------------------
    cbeam = []
    for i in range(16):
        seed = 9000 + i
        rng = np.random.default_rng(seed)
        phrases, V, c0, beta = gi.random_tree_spec(rng, max_phrases=12, max_len=5, max_vocab=16)
        _, tab = table_of(phrases, V, c0, beta)
        T = int(rng.integers(3, 14))
        lp = gi.random_emissions(rng, T, V)
        lam = float(rng.choice([0.0, 0.5, 1.0]))
        beam = int(rng.choice([2, 4, 8]))
        best, nbest = ctc_beam_boosted(EmissionMatrix(lp, blank_id=0), tab, DecodeConfig(lam=lam, beam_size=beam),
                                       want_trace=True)
        cbeam.append({"seed": seed, "V": V, "c0": c0, "beta": beta, "T": T, "lam": lam, "beam": beam,
                      "lp_sha": gi.sha(lp), "nbest": [res_dict(r) for r in nbest]})
    meta["ctc_beam"] = cbeam

    tgreedy, tbeam = [], []
    for i in range(16):
        seed = 9100 + i
        rng = np.random.default_rng(seed)
        phrases, V, c0, beta = gi.random_tree_spec(rng, max_phrases=10, max_len=4, max_vocab=12)
        _, tab = table_of(phrases, V, c0, beta)
        rows, default = gi.random_transducer_rows(rng, V)
        model = TableStepModel(flavor="transducer", default_row=default, rows=rows)
        T = int(rng.integers(2, 7))
        cap = int(rng.integers(1, 4))
        lam = float(rng.choice([0.0, 0.5, 1.0]))
        beam = int(rng.choice([2, 3, 4]))
        g = transducer_greedy_boosted(model, T, 0, tab, DecodeConfig(lam=lam, max_symbols_per_frame=cap),
                                      want_trace=True)
        best, nbest = transducer_beam_boosted(model, T, 0, tab,
                                              DecodeConfig(lam=lam, beam_size=beam, max_symbols_per_frame=cap),
                                              want_trace=True)
        case = {"seed": seed, "V": V, "c0": c0, "beta": beta, "T": T, "cap": cap, "lam": lam, "beam": beam,
                "rows_sha": gi.sha(default, *[rows[k] for k in sorted(rows)])}
        tgreedy.append({**case, "result": res_dict(g)})
        tbeam.append({**case, "nbest": [res_dict(r) for r in nbest]})
    meta["transducer_greedy"] = tgreedy
    meta["transducer_beam"] = tbeam

    aed = []
    for i in range(16):
        seed = 9200 + i
        rng = np.random.default_rng(seed)
        phrases, V, c0, beta = gi.random_tree_spec(rng, max_phrases=10, max_len=4, max_vocab=12)
        V = max(V, 4)
        _, tab = table_of(phrases, V, c0, beta)
        rows, default = gi.random_aed_rows(rng, V)
        eos = V - 1
        model = TableStepModel(flavor="aed", default_row=default, rows=rows, eos_id=eos)
        max_len = int(rng.integers(2, 6))
        lam = float(rng.choice([0.0, 0.5, 1.0]))
        beam = int(rng.choice([2, 3, 4]))
        bump = bool(i % 3 != 2)
        best, nbest = aed_beam_boosted(model, tab, DecodeConfig(lam=lam, beam_size=beam, eos_bump_enabled=bump),
                                       max_len=max_len, want_trace=True)
        aed.append({"seed": seed, "V": V, "c0": c0, "beta": beta, "eos": eos, "max_len": max_len, "lam": lam,
                    "beam": beam, "eos_bump": bump,
                    "rows_sha": gi.sha(default, *[rows[k] for k in sorted(rows)]),
                    "row_keys": sorted(rows), "nbest": [res_dict(r) for r in nbest]})
    meta["aed_beam"] = aed

    (HERE / "golden.json").write_text(json.dumps(meta, indent=1, sort_keys=True))
    np.savez_compressed(HERE / "golden.npz", **npz)
    print("wrote", HERE / "golden.json", HERE / "golden.npz")


if __name__ == "__main__":
    main()
