"""The C-ABI library loads and exports every symbol include/pgpb.h declares (CPU)."""

import ctypes
import re
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "pgpb.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pgpb_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    from paper_2508_07014_b200 import _lib

    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/pgpb.h but not exported"
    assert sorted(_lib.EXPORTED) == syms


def test_abi_version_and_error_channel():
    from paper_2508_07014_b200 import _lib

    assert _lib.abi_version() == 1
    rc = _lib.LIB.pgpb_trie_fail_links(0, None, None, 4, None)
    assert rc == _lib.PGPB_EINVAL
    assert "root" in _lib.last_error()


def test_library_is_sm100a():
    import subprocess

    from paper_2508_07014_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    assert "sm_100a" in out.stdout
