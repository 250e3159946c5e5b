"""Command-line surface (paper_2508_07014_b200/cli.py) vs the reference CLI.

tests/golden/cli_golden.json holds the reference CLI's exit codes, stdout and
written-table hashes for every command of tests/cli_workspace.py
(tests/golden/gen_cli_golden.py).  The workspace is rebuilt here with this
package's writers, whose bytes must equal the reference's; build-tree and
evaluate run on CPU, the decode commands need the GPU (every decoder is
bit-exact, so the JSON lines must be identical byte for byte).
"""

import contextlib
import hashlib
import io
import json
from functools import lru_cache
from pathlib import Path

import pytest

import cli_workspace as cw

HERE = Path(__file__).resolve().parent


@lru_cache(maxsize=1)
def golden():
    return json.loads((HERE / "golden" / "cli_golden.json").read_text())


class _Pkg:
    from paper_2508_07014_b200 import acoustic as _ac
    from paper_2508_07014_b200 import context as _cx

    Vocabulary = _cx.Vocabulary
    EmissionMatrix = _ac.EmissionMatrix
    TableStepModel = _ac.TableStepModel
    synth_ctc_emissions = staticmethod(_ac.synth_ctc_emissions)
    save_emissions = staticmethod(_ac.save_emissions)
    save_step_model = staticmethod(_ac.save_step_model)


def run(argv):
    from paper_2508_07014_b200.cli import main

    o, e = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(o), contextlib.redirect_stderr(e):
        rc = main(argv)
    return rc, o.getvalue(), e.getvalue()


@pytest.fixture(scope="module")
def ws(tmp_path_factory):
    root = tmp_path_factory.mktemp("cli") / "ws"
    w = cw.make_workspace(root, _Pkg)
    w["files_sha"] = {p.name: hashlib.sha256(p.read_bytes()).hexdigest() for p in sorted(root.iterdir())}
    cmds = cw.commands(w)
    for name in ("build", "build_uniform"):
        assert run(cmds[name])[0] == 0
    w["cmds"] = cmds
    return w


def _norm(text, ws):
    return text.replace(str(ws["root"]), "<WS>")


def test_workspace_files_are_byte_identical_to_reference_writers(ws):
    """TBT1 emissions, step-model JSON, vocab/context/refs files (the manifest
    embeds absolute scratch paths and is skipped)."""
    skip = {"manifest.jsonl"}
    ours = {k: v for k, v in ws["files_sha"].items() if k not in skip}
    ref = {k: v for k, v in golden()["_workspace_files_sha"].items() if k not in skip}
    assert ours == ref and len(ours) >= 15


@pytest.mark.parametrize("name", ["build", "build_uniform"])
def test_build_tree_matches_reference(ws, name):
    g = golden()[name]
    rc, out, err = run(ws["cmds"][name])
    assert rc == g["rc"] and out == g["stdout"] and _norm(err, ws) == g["stderr"]
    path = ws["cmds"][name][ws["cmds"][name].index("--out") + 1]
    assert hashlib.sha256(Path(path).read_bytes()).hexdigest() == g["table_sha"]


def test_evaluate_matches_reference(ws):
    g = golden()["evaluate"]
    rc, out, err = run(ws["cmds"]["evaluate"])
    assert (rc, out, _norm(err, ws)) == (g["rc"], g["stdout"], g["stderr"])


def test_usage_errors_exit_two(ws):
    v = str(ws["root"] / "vocab.txt")
    for argv in (["decode", "--mode", "ctc-greedy", "--vocab", v, "--emissions", str(ws["ems"][0])],  # no blank
                 ["decode", "--mode", "aed-beam", "--vocab", v, "--eos", "</s>", "--step-spec",
                  str(ws["root"] / "aed.json")],  # no max-len
                 ["decode", "--mode", "rnnt-greedy", "--vocab", v, "--blank", "<b>", "--step-spec",
                  str(ws["root"] / "rnnt.json")],  # no frames
                 ["decode", "--mode", "ctc-greedy", "--vocab", v, "--blank", "<b>", "--emissions",
                  str(ws["ems"][0]), "--manifest", str(ws["root"] / "manifest.jsonl")]):  # conflicting inputs
        with pytest.raises(SystemExit) as ei, contextlib.redirect_stderr(io.StringIO()):
            run(argv)
        assert ei.value.code == 2
    rc, _, err = run(["evaluate", "--refs", str(ws["root"] / "refs.jsonl"), "--hyps", str(ws["root"] / "nope.jsonl")])
    assert rc == 2 and err.startswith("error:")


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["ctc_greedy", "ctc_greedy_lam3", "ctc_greedy_plain", "ctc_beam", "rnnt_greedy",
                                  "rnnt_beam", "rnnt_spec", "rnnt_spec_beam", "aed", "aed_nobump", "manifest"])
def test_decode_output_byte_identical_to_reference(ws, name):
    g = golden()[name]
    rc, out, err = run(ws["cmds"][name])
    assert rc == g["rc"], err
    assert out == g["stdout"]


@pytest.mark.gpu
def test_bench_protocol(ws, tmp_path):
    argv = ["bench"] + ws["cmds"]["ctc_greedy"][1:] + ["--runs", "2", "--warmup", "1", "--out", str(tmp_path / "b.json")]
    rc, _, err = run(argv)
    assert rc == 0, err
    row = json.loads((tmp_path / "b.json").read_text())
    assert row["runs"] == 2 and len(row["times"]) == 2 and row["rtfx"] > 0 and row["audio_seconds"] > 0
