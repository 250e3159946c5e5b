"""Drop-in replacement for the reference's compiled module `phraseboost._kernels`.

Same two functions, same argument lists and return values as
/root/reference/pkg/src/phraseboost/_kernels.pyx (score_batch :30-72,
ctc_greedy :75-225): borrowed C-contiguous numpy inputs, fresh numpy
outputs.  Each call goes through the C-ABI host entry points of libpgpb
(H2D, sm_100a kernel, D2H).  Installing this module as
`phraseboost._backend._kernels` runs the reference's own code — and test
suite — on the B200 kernels.

A per-(arrays) device table cache avoids re-uploading the table for
repeated calls with the same arrays (the reference passes the same
ArcTable arrays on every decoding step).
"""

from __future__ import annotations

import threading

import numpy as np

from . import _lib

_DTYPES = {"int": np.int32, "float": np.float32}
_cache: dict = {}
_cache_lock = threading.Lock()


def _arr(x, kind: str, ndim: int = 1) -> np.ndarray:
    a = np.asarray(x)
    want = _DTYPES[kind]
    if a.dtype != want:
        raise ValueError(f"Buffer dtype mismatch, expected '{kind}' but got '{a.dtype}'")
    if a.ndim != ndim:
        raise ValueError(f"Buffer has wrong number of dimensions (expected {ndim}, got {a.ndim})")
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("ndarray is not C-contiguous")
    return a


class _ShimTable:
    def __init__(self, arrays, V):
        (arc_token, arc_to, arc_weight, state_start, state_end, backoff_to, backoff_weight,
         root_scores, root_next) = arrays
        S = state_start.shape[0]
        A = arc_token.shape[0]
        # The kernel module receives the dense root row, not unk_score: recover
        # it from a token with no root arc (all root rows are unk elsewhere).
        lo, hi = (int(state_start[0]), int(state_end[0])) if S else (0, 0)
        has_arc = np.zeros(V, bool)
        has_arc[arc_token[lo:hi]] = True
        free = np.flatnonzero(~has_arc)
        unk = float(root_scores[free[0]]) if free.size else 0.0
        h = _lib.c_void_p()
        fin = np.zeros(S, np.uint8)
        fs = np.zeros(S, np.float32)
        _lib.check(_lib.LIB.pgpb_table_create(
            S, V, A, _lib.ptr(arc_token), _lib.ptr(arc_to), _lib.ptr(arc_weight), _lib.ptr(state_start),
            _lib.ptr(state_end), _lib.ptr(backoff_to), _lib.ptr(backoff_weight), _lib.ptr(fin), _lib.ptr(fs),
            unk, _current_device(), _lib.ctypes.byref(h)), "pgpb_table_create")
        self.handle = h.value
        self._destroy = _lib.LIB.pgpb_table_destroy
        # the device table derives its root row from the arcs + unk score
        # (table.py:74-81); refuse a caller-supplied row that differs
        exp_s = np.full(V, np.float32(unk), np.float32)
        exp_n = np.zeros(V, np.int32)
        exp_s[arc_token[lo:hi]] = arc_weight[lo:hi]
        exp_n[arc_token[lo:hi]] = arc_to[lo:hi]
        if not (np.array_equal(exp_s.view(np.int32), root_scores.view(np.int32))
                and np.array_equal(exp_n, root_next)):
            raise ValueError("root row inconsistent with the arc table")

    def __del__(self):
        if getattr(self, "handle", None) and getattr(self, "_destroy", None) is not None:
            self._destroy(self.handle)


def _current_device() -> int:
    import torch

    _lib.require_cuda()
    return torch.cuda.current_device()


def _table(arrays, V) -> _ShimTable:
    key = tuple((a.ctypes.data, a.shape[0]) for a in arrays) + (V,)
    with _cache_lock:
        t = _cache.get(key)
        if t is not None and all(np.shares_memory(a, b) for a, b in zip(arrays, t[0])):
            return t[1]
        st = _ShimTable(arrays, V)
        if len(_cache) > 64:
            _cache.clear()
        _cache[key] = (arrays, st)
        return st


def score_batch(arc_token, arc_to, arc_weight, state_start, state_end, backoff_to, backoff_weight,
                root_scores, root_next, states):
    """_kernels.pyx:30-72: (scores float32[B,V], next int32[B,V])."""
    arrays = [_arr(arc_token, "int"), _arr(arc_to, "int"), _arr(arc_weight, "float"), _arr(state_start, "int"),
              _arr(state_end, "int"), _arr(backoff_to, "int"), _arr(backoff_weight, "float"),
              _arr(root_scores, "float"), _arr(root_next, "int")]
    st = _arr(states, "int")
    V = arrays[7].shape[0]
    B = st.shape[0]
    scores = np.empty((B, V), np.float32)
    nxt = np.empty((B, V), np.int32)
    if B:
        t = _table(arrays, V)
        _lib.check(_lib.LIB.pgpb_advance_host(t.handle, _lib.ptr(st), B, _lib.ptr(scores), _lib.ptr(nxt),
                                              _lib.stream_ptr()), "pgpb_advance_host")
    return scores, nxt


def ctc_greedy(logprobs, blank, lam, use_boost, arc_token, arc_to, arc_weight, state_start, state_end,
               backoff_to, backoff_weight, root_scores, root_next):
    """_kernels.pyx:75-225: (tokens int32[n], am, boost, deltas float64[n], states int32[n])."""
    lp = np.asarray(logprobs)
    if lp.dtype != np.float32:
        raise ValueError(f"Buffer dtype mismatch, expected 'float' but got '{lp.dtype}'")
    if lp.ndim != 2:
        raise ValueError(f"Buffer has wrong number of dimensions (expected 2, got {lp.ndim})")
    if not lp.flags["C_CONTIGUOUS"]:
        raise ValueError("ndarray is not C-contiguous")
    T, V = lp.shape
    handle = None
    if use_boost:
        arrays = [_arr(arc_token, "int"), _arr(arc_to, "int"), _arr(arc_weight, "float"), _arr(state_start, "int"),
                  _arr(state_end, "int"), _arr(backoff_to, "int"), _arr(backoff_weight, "float"),
                  _arr(root_scores, "float"), _arr(root_next, "int")]
        handle = _table(arrays, V).handle
    else:
        _current_device()
    tok = np.empty(max(T, 1), np.int32)
    dl = np.empty(max(T, 1), np.float64)
    stt = np.empty(max(T, 1), np.int32)
    n = _lib.c_int64()
    am = _lib.c_double()
    bo = _lib.c_double()
    _lib.check(_lib.LIB.pgpb_ctc_greedy_host(
        handle, _lib.ptr(lp), T, V, int(blank), float(lam), int(bool(use_boost)), _lib.ptr(tok), _lib.ptr(dl),
        _lib.ptr(stt), _lib.ctypes.byref(n), _lib.ctypes.byref(am), _lib.ctypes.byref(bo), _lib.stream_ptr()),
        "pgpb_ctc_greedy_host")
    k = n.value
    return tok[:k].copy(), am.value, bo.value, dl[:k].copy(), stt[:k].copy()
