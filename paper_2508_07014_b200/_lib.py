"""ctypes binding of the C-ABI library libpgpb.so (include/pgpb.h).

The product path has no CPU fallback: importing this module on a machine
where libpgpb.so is missing raises immediately, and every compute entry
point needs a CUDA device.  Error codes from the library are mapped to the
reference's exception types (ValueError / IndexError / TableFormatError).
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_float, c_int32, c_int64, c_uint8, c_void_p
from pathlib import Path

import numpy as np

from .errors import TableFormatError

LIB_PATH = Path(os.environ.get("PGPB_LIB_PATH") or Path(__file__).resolve().parent / "libpgpb.so")

PGPB_OK = 0
PGPB_EINVAL = -1
PGPB_ERANGE = -2
PGPB_ECUDA = -3
PGPB_ENOMEM = -4
PGPB_EFORMAT = -5


class TableInfo(ctypes.Structure):
    _fields_ = [
        ("num_states", c_int32),
        ("vocab_size", c_int32),
        ("num_arcs", c_int32),
        ("max_chain", c_int32),
        ("closure_entries", c_int64),
        ("max_closure", c_int32),
        ("device", c_int32),
        ("device_bytes", c_int64),
        ("unk_score", c_float),
        ("max_root_score", c_float),
    ]


class LabelLoopState(ctypes.Structure):
    """pgpb_label_loop_state (include/pgpb.h)."""

    _fields_ = [(n, c_void_p) for n in ("t", "k", "lengths", "n", "last", "tree", "am", "boost", "tokens",
                                         "deltas", "states")] + [("lmax", c_int64), ("cap", c_int32),
                                                                 ("durations", c_void_p), ("tree_off", c_void_p)]


class BeamHyps(ctypes.Structure):
    """pgpb_beam_hyps (include/pgpb.h): [B, K] struct of arrays."""

    _fields_ = [(n, c_void_p) for n in ("am", "boost", "tree", "last", "node", "len", "hash", "flags", "parent")]


class BeamTrace(ctypes.Structure):
    """pgpb_beam_trace: append-only per-utterance trie of trace steps."""

    _fields_ = [(n, c_void_p) for n in ("parent", "token", "state", "delta", "count", "overflow")] + \
        [("nmax", c_int64)]


class TBeamState(ctypes.Structure):
    """pgpb_tbeam_state."""

    _fields_ = [("hyps", BeamHyps), ("pool", BeamHyps), ("pool_count", c_void_p), ("trace", BeamTrace),
                ("t", c_void_p), ("lengths", c_void_p), ("beam", c_int32), ("cap", c_int32), ("pool_cap", c_int32),
                ("rollback", c_int32)]


class AedState(ctypes.Structure):
    """pgpb_aed_state."""

    _fields_ = [("hyps", BeamHyps), ("trace", BeamTrace), ("row_max", c_void_p), ("any_active", c_void_p),
                ("beam", c_int32), ("max_len", c_int32), ("eos", c_int32), ("eos_bump", c_int32),
                ("rollback", c_int32)]


class AedGreedyState(ctypes.Structure):
    """pgpb_aed_greedy_state."""

    _fields_ = [("tree", c_void_p), ("am", c_void_p), ("boost", c_void_p), ("len", c_void_p), ("ended", c_void_p),
                ("feed", c_void_p), ("tokens", c_void_p), ("deltas", c_void_p), ("states", c_void_p),
                ("row_max", c_void_p), ("final_bonus", c_void_p), ("any_active", c_void_p),
                ("max_len", c_int32), ("eos", c_int32), ("rollback", c_int32)]


class CtcBeamOut(ctypes.Structure):
    """pgpb_ctc_beam_out."""

    _fields_ = [("pb", c_void_p), ("pnb", c_void_p), ("boost", c_void_p), ("tree", c_void_p), ("len", c_void_p),
                ("node", c_void_p), ("count", c_void_p), ("trace_parent", c_void_p), ("trace_token", c_void_p),
                ("trace_state", c_void_p), ("trace_delta", c_void_p), ("trace_nmax", c_int64),
                ("overflow", c_void_p)]


# name -> argtypes (all return int unless listed in _VOID / _OTHER)
_P = c_void_p
_SIGS = {
    "pgpb_abi_version": [],
    "pgpb_set_tuning": [ctypes.c_char_p, c_int32],
    "pgpb_trie_build": [_P, _P, c_int64, c_int32, c_double, c_double, c_int32, c_double, c_int64,
                        _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "pgpb_trie_fail_links": [c_int64, _P, _P, c_int32, _P],
    "pgpb_trie_compile": [c_int64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "pgpb_table_create": [c_int32, c_int32, c_int32, _P, _P, _P, _P, _P, _P, _P, _P, _P, c_float,
                          c_int32, POINTER(c_void_p)],
    "pgpb_table_info_get": [c_void_p, POINTER(TableInfo)],
    "pgpb_table_load_gpb1": [_P, c_int64, c_int32, POINTER(c_void_p)],
    "pgpb_table_load_gpb1_file": [ctypes.c_char_p, c_int32, POINTER(c_void_p)],
    "pgpb_advance": [c_void_p, _P, c_int64, _P, _P, c_void_p],
    "pgpb_advance_host": [c_void_p, _P, c_int64, _P, _P, c_void_p],
    "pgpb_advance_chain": [c_void_p, _P, c_int64, _P, _P, c_void_p],
    "pgpb_advance_steps": [c_void_p, _P, _P, c_int32, c_int64, _P, _P, _P, _P, c_int32, c_void_p],
    "pgpb_ctc_greedy": [c_void_p, _P, c_int64, c_int64, c_int32, _P, c_int32, c_double, c_int32,
                        _P, _P, _P, _P, _P, _P, c_void_p],
    "pgpb_ctc_greedy_host": [c_void_p, _P, c_int64, c_int32, c_int32, c_double, c_int32, _P, _P, _P,
                             _P, _P, _P, c_void_p],
    "pgpb_greedy_step": [c_void_p, _P, c_int64, c_int64, c_int32, _P, _P, c_int32, c_double, c_int32,
                         _P, _P, _P, _P, _P, c_void_p],
    "pgpb_row_max": [c_void_p, _P, c_void_p],
    "pgpb_final_bonus": [c_void_p, _P, c_void_p],
    "pgpb_backoff_total": [c_void_p, _P, c_void_p],
    "pgpb_label_loop_step": [c_void_p, _P, c_int64, c_int64, c_int32, c_int32, c_double, c_int32,
                             POINTER(LabelLoopState), _P, _P, _P, c_void_p],
    "pgpb_label_loop_step_logits": [c_void_p, _P, c_int64, _P, c_int64, c_int32, c_int32, c_double, c_int32,
                                    POINTER(LabelLoopState), _P, _P, _P, c_void_p],
    "pgpb_rnnt_joint_hidden": [_P, c_int64, c_int32, _P, _P, _P, c_int64, _P, c_int64, c_void_p],
    "pgpb_rnnt_beam_hidden": [_P, c_int64, c_int32, _P, _P, _P, _P, c_int64, c_int32, c_int32, _P, c_void_p],
    "pgpb_rnnt_lstm_update": [_P, _P, _P, c_int64, _P, _P, _P, c_int64, c_int32, c_void_p],
    "pgpb_beam_topk": [c_void_p, _P, c_int64, c_int64, c_int32, c_int32, c_int32, _P, _P, _P, _P,
                       _P, _P, _P, c_double, c_int32, c_int32, _P, _P, _P, _P, _P, _P, c_void_p],
    "pgpb_tbeam_wave": [c_void_p, _P, c_int64, c_int64, c_int32, c_int32, c_double, c_int32, c_int32,
                        POINTER(TBeamState), c_void_p],
    "pgpb_tbeam_wave_fused": [c_void_p, _P, c_int64, _P, c_int64, c_int64, c_int32, c_int32, c_double, c_int32,
                              c_int32, POINTER(TBeamState), _P, c_int64, c_int32, _P, _P, c_void_p],
    "pgpb_phrase_hits": [c_void_p, _P, _P, c_int64, _P, _P, _P, _P, _P, _P, c_void_p],
    "pgpb_aed_step": [c_void_p, _P, c_int64, c_int64, c_int32, c_double, c_int32, POINTER(AedState), c_void_p],
    "pgpb_ctc_beam": [c_void_p, _P, c_int64, c_int64, c_int32, _P, c_int32, c_int32, c_double, c_int32,
                      POINTER(CtcBeamOut), c_void_p],
    "pgpb_aed_greedy_step": [c_void_p, _P, c_int64, c_int64, c_int32, c_double, c_int32, POINTER(AedGreedyState),
                             c_void_p],
}

# Every symbol include/pgpb.h declares (checked by tests/test_abi.py).
EXPORTED = sorted(list(_SIGS) + ["pgpb_last_error", "pgpb_table_destroy"])


def _load() -> ctypes.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA extension first "
            "(python __graft_entry__.py or python paper_2508_07014_b200/_build.py); there is no CPU fallback"
        )
    lib = ctypes.CDLL(str(LIB_PATH))
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = c_int32
    lib.pgpb_last_error.argtypes = []
    lib.pgpb_last_error.restype = ctypes.c_char_p
    lib.pgpb_table_destroy.argtypes = [c_void_p]
    lib.pgpb_table_destroy.restype = None
    return lib


LIB = _load()


def last_error() -> str:
    msg = LIB.pgpb_last_error()
    return msg.decode("utf-8", "replace") if msg else ""


def check(rc: int, what: str = "") -> None:
    """Raise the reference-equivalent exception for a library error code."""
    if rc == PGPB_OK:
        return
    msg = last_error() or what
    if rc == PGPB_ERANGE:
        raise IndexError(msg)
    if rc == PGPB_EINVAL:
        raise ValueError(msg)
    if rc == PGPB_EFORMAT:
        raise TableFormatError(msg)
    if rc == PGPB_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"pgpb CUDA error: {msg}")


def ptr(a) -> int | None:
    """Data pointer of a contiguous numpy array or torch tensor (None if None)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("ndarray is not C-contiguous")
        return a.ctypes.data
    if not a.is_contiguous():
        raise ValueError("tensor is not contiguous")
    return a.data_ptr()


def stream_ptr(stream=None) -> int:
    """cudaStream_t of `stream` (or torch's current stream) as an int."""
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def require_cuda() -> None:
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_2508_07014_b200 needs a CUDA device (sm_100a); there is no CPU fallback"
        )


def set_tuning(key: str, value: int) -> None:
    """Code-path override (pgpb_set_tuning); 0 = automatic.  Tests only."""
    check(LIB.pgpb_set_tuning(key.encode(), int(value)), "pgpb_set_tuning")


def abi_version() -> int:
    return int(LIB.pgpb_abi_version())
