"""Backend reporting, mirroring the reference's `phraseboost._backend`
(/root/reference/pkg/src/phraseboost/_backend.py:27-53).

There is exactly one backend here — the sm_100a CUDA kernels in
libpgpb.so — so there is nothing to select: `backend_name()` is "cuda",
`kernels()` returns the kernel module with the reference's `_kernels`
signatures (kernels_shim), and forcing the reference's "python" backend is
refused rather than silently falling back to CPU code.
"""

from __future__ import annotations

import os
from contextlib import contextmanager

from . import _lib  # noqa: F401  (fails loudly when libpgpb.so is missing)

_env = os.environ.get("PHRASEBOOST_BACKEND", "").strip().lower()
if _env not in ("", "compiled", "cuda"):
    raise RuntimeError(f"PHRASEBOOST_BACKEND={_env!r}: this build only has the CUDA backend")

HAVE_COMPILED = True


def compiled_active() -> bool:
    return True


def backend_name() -> str:
    return "cuda"


def kernels():
    """Module exposing score_batch / ctc_greedy with the reference signatures."""
    from . import kernels_shim

    return kernels_shim


@contextmanager
def forced_backend(name: str):
    if name not in ("python", "compiled", "cuda"):
        raise ValueError(f"unknown backend {name!r}")
    if name == "python":
        raise RuntimeError("no CPU backend: every score runs on the GPU")
    yield
