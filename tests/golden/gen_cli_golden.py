"""Record the REFERENCE CLI's outputs on the deterministic workspace of
tests/cli_workspace.py (run in the build container, needs /root/reference):

    python tests/golden/gen_cli_golden.py

Builds the reference package in a scratch copy (as gen_golden.py does),
writes the workspace with the reference's own writers, runs
phraseboost.cli.main for every command and stores exit code, stdout and
the sha256 of written tables in tests/golden/cli_golden.json.
"""

from __future__ import annotations

import contextlib
import hashlib
import io
import json
import sys
import tempfile
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE))

import cli_workspace as cw  # noqa: E402
from gen_golden import ensure_ref  # noqa: E402


def main():
    sys.path.insert(0, str(ensure_ref(None)))
    import phraseboost.acoustic as ac
    import phraseboost.context as cx
    from phraseboost.cli import main as ref_main

    class Pkg:
        Vocabulary = cx.Vocabulary
        EmissionMatrix = ac.EmissionMatrix
        TableStepModel = ac.TableStepModel
        synth_ctc_emissions = staticmethod(ac.synth_ctc_emissions)
        save_emissions = staticmethod(ac.save_emissions)
        save_step_model = staticmethod(ac.save_step_model)

    out = {}
    with tempfile.TemporaryDirectory() as d:
        root = Path(d) / "ws"
        ws = cw.make_workspace(root, Pkg)
        files = {p.name: hashlib.sha256(p.read_bytes()).hexdigest() for p in sorted(root.iterdir())}
        for name, argv in cw.commands(ws).items():
            buf_o, buf_e = io.StringIO(), io.StringIO()
            with contextlib.redirect_stdout(buf_o), contextlib.redirect_stderr(buf_e):
                rc = ref_main(argv)
            rec = {"rc": rc, "stdout": buf_o.getvalue().replace(str(root), "<WS>"),
                   "stderr": buf_e.getvalue().replace(str(root), "<WS>")}
            if name.startswith("build"):
                rec["table_sha"] = hashlib.sha256(Path(argv[argv.index("--out") + 1]).read_bytes()).hexdigest()
            out[name] = rec
    out["_workspace_files_sha"] = files
    (HERE / "cli_golden.json").write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
    print("wrote", HERE / "cli_golden.json", len(out) - 1, "commands")


if __name__ == "__main__":
    main()
