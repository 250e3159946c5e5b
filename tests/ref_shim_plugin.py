"""pytest plugin: run the REFERENCE's own test suites on the B200 kernels.

Loaded with `-p ref_shim_plugin` when pytest runs inside the reference
package copy (baseline/_ref/pkg, made by __graft_entry__.build()).  Before
collection it installs paper_2508_07014_b200.kernels_shim as the
reference's compiled kernel module — the binding a maintainer would add at
/root/reference/pkg/src/phraseboost/_backend.py:13-16 —
so every `_backend.kernels()` call (table.py:200-213, decoding.py:170-191)
reaches libpgpb's sm_100a kernels through the C-ABI.  At the end it prints
how many shim calls ran, so a pass cannot come from the NumPy backend alone.
"""

from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

_calls = {"score_batch": 0, "ctc_greedy": 0}


def pytest_configure(config):
    if str(ROOT) not in sys.path:
        sys.path.insert(0, str(ROOT))
    src = Path.cwd() / "src"
    if src.is_dir() and str(src) not in sys.path:
        sys.path.insert(0, str(src))
    import phraseboost._backend as be

    from paper_2508_07014_b200 import kernels_shim

    class _Counted:
        """kernels_shim with call counters (same functions, same signatures)."""

        @staticmethod
        def score_batch(*a, **k):
            _calls["score_batch"] += 1
            return kernels_shim.score_batch(*a, **k)

        @staticmethod
        def ctc_greedy(*a, **k):
            _calls["ctc_greedy"] += 1
            return kernels_shim.ctc_greedy(*a, **k)

    be._kernels = _Counted
    be.HAVE_COMPILED = True


def pytest_terminal_summary(terminalreporter):
    terminalreporter.write_line(f"B200 shim calls: score_batch={_calls['score_batch']} "
                                f"ctc_greedy={_calls['ctc_greedy']}")
