"""Deterministic CLI workspace (vocab, context, TBT1 emissions, manifest,
step-model specs, refs/hyps) and the command list shared by the golden
generator (tests/golden/gen_cli_golden.py, run against the reference CLI)
and tests/test_cli.py (run against ours).  Files are written with this
package's writers, which follow the reference formats byte for byte."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

LETTERS = "abcdefghijklmnopqrstuvwxyz"
PHRASES = ["cat", "cats", "csv", "sit", "sat", "act", "tic", "a"]


def _log_softmax(x):
    m = x.max(axis=-1, keepdims=True)
    return x - (m + np.log(np.exp(x - m).sum(axis=-1, keepdims=True)))


def make_workspace(root: Path, pkg) -> dict:
    """pkg: the module providing Vocabulary/synth_ctc_emissions/save_* (ours or the reference's)."""
    root.mkdir(parents=True, exist_ok=True)
    tokens = ("<b>",) + tuple(LETTERS) + ("</s>",)
    (root / "vocab.txt").write_text("\n".join(tokens) + "\n")
    (root / "context.txt").write_text("\n".join(PHRASES) + "\n")
    vocab = pkg.Vocabulary(tokens=tokens, blank_id=0, eos_id=27)
    V = len(tokens)
    pool = [vocab.id_of(ch) for ch in "qxzjk"]
    ems = []
    words = ["cat", "sit", "cats", "tic tac", "act sat", "csv"]
    for i, w in enumerate(words):
        target = [vocab.id_of(ch) for ch in w.replace(" ", "")]
        em = pkg.synth_ctc_emissions(target, vocab, 0.5 + 0.25 * (i % 3), seed=100 + i, distractor_pool=pool,
                                     blanks_between=1 + (i % 3))
        p = root / f"utt{i}.tbt"
        pkg.save_emissions(em, p)
        ems.append(p)
    rng = np.random.default_rng(7)
    for i in range(3):
        lp = _log_softmax(rng.normal(0.0, 2.0, size=(int(rng.integers(5, 40)), V))).astype(np.float32)
        p = root / f"rand{i}.tbt"
        pkg.save_emissions(pkg.EmissionMatrix(lp, blank_id=0), p)
        ems.append(p)
    with open(root / "manifest.jsonl", "w") as fh:
        for k in (2, 0, 5):
            fh.write(json.dumps({"id": f"m{k}", "emissions": str(ems[k])}) + "\n")

    def row(**kw):
        logits = np.full(V, -9.0)
        for k, v in kw.items():
            logits[int(k)] = v
        return _log_softmax(logits).astype(np.float32)

    c, a, t, s = (vocab.id_of(ch) for ch in "cats")
    rnnt = pkg.TableStepModel(flavor="transducer", default_row=row(**{"0": 3.0, str(s): 1.0}),
                              rows={"": row(**{str(c): 2.0}), str(c): row(**{str(a): 2.0, "0": 1.5}),
                                    str(a): row(**{str(t): 2.0, str(s): 1.8})})
    pkg.save_step_model(rnnt, root / "rnnt.json")
    aed = pkg.TableStepModel(flavor="aed", default_row=row(**{"27": 2.0, str(s): 1.9}),
                             rows={"": row(**{str(c): 3.0, str(s): 2.5}), str(c): row(**{str(a): 3.0}),
                                   f"{c},{a}": row(**{str(t): 3.0, "27": 2.9})}, eos_id=27)
    pkg.save_step_model(aed, root / "aed.json")
    refs = ["the cat sat", "a csv file", "tic tac toe", "cats sit"]
    hyps = ["the cat sit", "a csv file", "tic toe", "cat sit"]
    (root / "refs.jsonl").write_text("".join(json.dumps({"id": f"u{i}", "text": r}) + "\n" for i, r in enumerate(refs)))
    (root / "hyps.jsonl").write_text("".join(json.dumps({"id": f"u{i}", "text": h}) + "\n" for i, h in enumerate(hyps)))
    return {"root": root, "ems": ems}


def commands(ws: dict) -> dict:
    """name -> argv (paths relative to the workspace root are resolved here)."""
    r = ws["root"]
    ems = [str(p) for p in ws["ems"]]
    v, tab, tab_u = str(r / "vocab.txt"), str(r / "table.gpb"), str(r / "table_u.gpb")
    ctc = ["--vocab", v, "--blank", "<b>"]
    return {
        "build": ["build-tree", "--vocab", v, "--context", str(r / "context.txt"), "--out", tab],
        "build_uniform": ["build-tree", "--vocab", v, "--context", str(r / "context.txt"), "--out", tab_u,
                          "--weight-mode", "uniform", "--final-bonus", "0.5", "--unk-score", "-0.5",
                          "--min-chars", "1"],
        "ctc_greedy": ["decode", "--mode", "ctc-greedy", *ctc, "--table", tab, "--trace", "--emissions", *ems],
        "ctc_greedy_lam3": ["decode", "--mode", "ctc-greedy", *ctc, "--table", tab_u, "--lambda", "3",
                            "--emissions", *ems],
        "ctc_greedy_plain": ["decode", "--mode", "ctc-greedy", *ctc, "--emissions", *ems],
        "ctc_beam": ["decode", "--mode", "ctc-beam", *ctc, "--table", tab, "--beam", "4", "--trace",
                     "--emissions", *ems[:6]],
        "rnnt_greedy": ["decode", "--mode", "rnnt-greedy", *ctc, "--table", tab, "--max-symbols", "1",
                        "--trace", "--emissions", *ems[:4]],
        "rnnt_beam": ["decode", "--mode", "rnnt-beam", *ctc, "--table", tab, "--max-symbols", "1", "--beam", "3",
                      "--emissions", *ems[:4]],
        "rnnt_spec": ["decode", "--mode", "rnnt-greedy", *ctc, "--table", tab, "--step-spec",
                      str(r / "rnnt.json"), "--frames", "6", "--max-symbols", "2", "--trace"],
        "rnnt_spec_beam": ["decode", "--mode", "rnnt-beam", *ctc, "--table", tab, "--step-spec",
                           str(r / "rnnt.json"), "--frames", "5", "--max-symbols", "2", "--beam", "4"],
        "aed": ["decode", "--mode", "aed-beam", "--vocab", v, "--eos", "</s>", "--table", tab, "--step-spec",
                str(r / "aed.json"), "--max-len", "8", "--trace"],
        "aed_nobump": ["decode", "--mode", "aed-beam", "--vocab", v, "--eos", "</s>", "--table", tab,
                       "--step-spec", str(r / "aed.json"), "--max-len", "6", "--no-eos-bump", "--beam", "2"],
        "manifest": ["decode", "--mode", "ctc-greedy", *ctc, "--table", tab, "--manifest",
                     str(r / "manifest.jsonl")],
        "evaluate": ["evaluate", "--refs", str(r / "refs.jsonl"), "--hyps", str(r / "hyps.jsonl"), "--context",
                     str(r / "context.txt")],
    }


GPU_FREE = ("build", "build_uniform", "evaluate")
