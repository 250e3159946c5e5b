"""The reference's own test suites, unchanged, on the B200 kernels.

SURVEY §8(b) parity shim / §7 gate (i): pytest runs inside the copy of the
reference package that __graft_entry__.build() places in baseline/_ref/pkg
(git-ignored; it travels to the GPU box with the snapshot), with
tests/ref_shim_plugin.py installing kernels_shim as
`phraseboost._backend._kernels`.  The suites compare the compiled backend
(now: libpgpb through the C-ABI) against the reference's NumPy backend and
its golden known answers (test_backends.py:47-78, test_table.py:153-168,
:314-343, test_acceptance.py:47-441, test_decoding.py)."""

import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref" / "pkg"

pytestmark = pytest.mark.gpu

# every reference suite that reaches the kernel module (score_batch /
# ctc_greedy): the table, backend, acceptance and decoder suites, and the
# CLI suite that decodes through the same calls
SUITES = ["test_table.py", "test_backends.py", "test_acceptance.py", "test_decoding.py", "test_cli.py"]


@pytest.mark.skipif(not (REF / "tests").is_dir(), reason="baseline/_ref/pkg not built (run __graft_entry__.build())")
@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_passes_on_b200_kernels(suite):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(ROOT / "tests"), str(ROOT), str(REF / "src"),
                                         env.get("PYTHONPATH", "")])
    env.pop("PHRASEBOOST_BACKEND", None)
    r = subprocess.run([sys.executable, "-m", "pytest", "-p", "ref_shim_plugin", "-q", "-p", "no:cacheprovider",
                        f"tests/{suite}"], cwd=REF, env=env, capture_output=True, text=True, timeout=1500)
    tail = "\n".join((r.stdout + r.stderr).splitlines()[-25:])
    assert r.returncode == 0, tail
    m = re.search(r"(\d+) passed", r.stdout)
    assert m and int(m.group(1)) > 0, tail
    calls = re.search(r"B200 shim calls: score_batch=(\d+) ctc_greedy=(\d+)", r.stdout)
    assert calls and int(calls.group(1)) + int(calls.group(2)) > 0, "the suite never reached the B200 kernels"
    assert "skipped" not in r.stdout.splitlines()[-1] or suite != "test_backends.py", tail
