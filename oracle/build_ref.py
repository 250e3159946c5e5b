"""Compile the reference's own Cython kernel module into oracle/_ref/.

ORACLE / TEST INFRASTRUCTURE ONLY.  Builds
/root/reference/pkg/src/phraseboost/_kernels.pyx (the reference's compiled
hot path, _kernels.pyx:30-225) exactly as the reference's setup.py does
(Cython -> C, gcc -O3, numpy headers, pkg/setup.py:4-17), writing only into
oracle/_ref/.  The reference sources are read in place and never copied into
the repository; oracle/_ref/ is git-ignored and travels to the GPU box as a
built artefact so bench.py can time the reference's own CPU kernels there.
"""

from __future__ import annotations

import argparse
import subprocess
import sys
import sysconfig
from pathlib import Path

HERE = Path(__file__).resolve().parent
OUT = HERE / "_ref"


def build(pyx: Path) -> Path:
    import numpy as np

    if not pyx.exists():
        raise FileNotFoundError(pyx)
    OUT.mkdir(exist_ok=True)
    c_file = OUT / "_kernels.c"
    subprocess.run(
        [sys.executable, "-m", "cython", "-3", "-o", str(c_file), str(pyx)], check=True
    )
    suffix = sysconfig.get_config_var("EXT_SUFFIX")
    so = OUT / f"_kernels{suffix}"
    cmd = [
        "gcc", "-O3", "-shared", "-fPIC", "-fwrapv",
        f"-I{sysconfig.get_paths()['include']}", f"-I{np.get_include()}",
        "-DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION", str(c_file), "-o", str(so), "-lm",
    ]
    subprocess.run(cmd, check=True)
    c_file.unlink()
    return so


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--pyx", default="/root/reference/pkg/src/phraseboost/_kernels.pyx")
    print(build(Path(ap.parse_args().pyx)))
