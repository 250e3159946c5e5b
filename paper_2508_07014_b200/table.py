"""Flat arc table (tree compilation, stage 2) and the GPU advance.

API mirror of the reference's `phraseboost.table`
(/root/reference/pkg/src/phraseboost/table.py):

* `ArcTable` (:53-127) — the same twelve arrays (CSR sorted by
  (from, token), per-state backoff, finals, dense root row), plus a lazily
  created device copy per GPU (`device_table()`), which holds the packed
  16-byte records and the flattened backoff closure.
* `compile_arc_table` (:138-187) — native (libpgpb, csrc/pgpb_tree.cpp).
* `get_scores_batch` (:190-214) / `advance` — the advance kernel.  numpy /
  list input returns numpy (the reference's contract, through the C-ABI
  host entry point); a CUDA tensor returns CUDA tensors without a host
  round trip.
* `naive_score` (:217-247), GPB1 `save_table` / `load_table` (:250-310),
  `state_strings` (:313-333).
"""

from __future__ import annotations

import struct
import threading
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import _lib
from .context import Vocabulary
from .errors import TableFormatError
from .tree import PrefixTree

MAGIC = b"GPB1"
VERSION = 1
_HEADER = struct.Struct("<4sIIIIf")


class _DeviceTable:
    """Owner of one pgpb_table handle (device copy of an ArcTable)."""

    def __init__(self, table: "ArcTable", device: int):
        h = _lib.c_void_p()
        c = np.ascontiguousarray
        self._keep = [
            c(table.arc_token, np.int32), c(table.arc_to, np.int32), c(table.arc_weight, np.float32),
            c(table.state_start, np.int32), c(table.state_end, np.int32), c(table.backoff_to, np.int32),
            c(table.backoff_weight, np.float32), c(table.is_final, np.uint8), c(table.final_score, np.float32),
        ]
        k = self._keep
        _lib.check(_lib.LIB.pgpb_table_create(
            table.num_states, table.vocab_size, table.num_arcs, *[_lib.ptr(a) for a in k],
            float(table.unk_score), int(device), _lib.ctypes.byref(h),
        ), "pgpb_table_create")
        self.handle = h.value
        self.device = device
        self._keep = None
        self._row_max = None
        self._final = None
        self._bt = None
        self._destroy = _lib.LIB.pgpb_table_destroy  # survives interpreter teardown

    @classmethod
    def _from_handle(cls, handle: int, device: int) -> "_DeviceTable":
        d = cls.__new__(cls)
        d.handle, d.device, d._keep, d._row_max, d._final, d._bt = handle, device, None, None, None, None
        d._destroy = _lib.LIB.pgpb_table_destroy
        return d

    def info(self) -> _lib.TableInfo:
        out = _lib.TableInfo()
        _lib.check(_lib.LIB.pgpb_table_info_get(self.handle, _lib.ctypes.byref(out)))
        return out

    def row_max(self):
        """max_v score[s, v] per state as a CUDA f32 tensor (cached)."""
        import torch

        if self._row_max is None:
            out = torch.empty(self.info().num_states, dtype=torch.float32, device=f"cuda:{self.device}")
            _lib.check(_lib.LIB.pgpb_row_max(self.handle, out.data_ptr(), _lib.stream_ptr()))
            self._row_max = out
        return self._row_max

    def final_bonus(self):
        """final_score[s] on final states, 0 elsewhere, as a CUDA f32 tensor
        (cached): the final part of the AED eos bump (decoding.py:546-552)."""
        import torch

        if self._final is None:
            out = torch.empty(self.info().num_states, dtype=torch.float32, device=f"cuda:{self.device}")
            _lib.check(_lib.LIB.pgpb_final_bonus(self.handle, out.data_ptr(), _lib.stream_ptr()))
            self._final = out
        return self._final

    def backoff_total(self):
        """Per state the fp32 backoff total of its chain (the rollback
        extension's credit), as a CUDA f32 tensor (cached)."""
        import torch

        if self._bt is None:
            out = torch.empty(self.info().num_states, dtype=torch.float32, device=f"cuda:{self.device}")
            _lib.check(_lib.LIB.pgpb_backoff_total(self.handle, out.data_ptr(), _lib.stream_ptr()))
            self._bt = out
        return self._bt

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and getattr(self, "_destroy", None) is not None:
            self._destroy(h)
            self.handle = None


@dataclass
class ArcTable:
    """Compiled boosting automaton; state 0 is the root (table.py:53-81)."""

    num_states: int
    vocab_size: int
    arc_from: np.ndarray
    arc_token: np.ndarray
    arc_to: np.ndarray
    arc_weight: np.ndarray
    state_start: np.ndarray
    state_end: np.ndarray
    backoff_to: np.ndarray
    backoff_weight: np.ndarray
    is_final: np.ndarray
    final_score: np.ndarray
    unk_score: float = 0.0
    root_scores: np.ndarray = field(init=False, repr=False)
    root_next: np.ndarray = field(init=False, repr=False)

    def __post_init__(self):
        V = self.vocab_size
        rs = np.full(V, np.float32(self.unk_score), dtype=np.float32)
        rn = np.zeros(V, dtype=np.int32)
        lo, hi = int(self.state_start[0]), int(self.state_end[0])
        rs[self.arc_token[lo:hi]] = self.arc_weight[lo:hi]
        rn[self.arc_token[lo:hi]] = self.arc_to[lo:hi]
        self.root_scores = rs
        self.root_next = rn
        self._dev: dict[int, _DeviceTable] = {}
        self._dev_lock = threading.Lock()

    @property
    def num_arcs(self) -> int:
        return int(self.arc_from.shape[0])

    def validate(self) -> None:
        """Every structural invariant of table.py:87-127, vectorised."""
        S, V, A = self.num_states, self.vocab_size, self.num_arcs
        if S < 1 or V < 1:
            raise TableFormatError(f"need at least 1 state and 1 token, got S={S} V={V}")
        for name in ("arc_from", "arc_token", "arc_to", "arc_weight"):
            if getattr(self, name).shape != (A,):
                raise TableFormatError(f"{name} length != num_arcs")
        for name in ("state_start", "state_end", "backoff_to", "backoff_weight", "is_final", "final_score"):
            if getattr(self, name).shape != (S,):
                raise TableFormatError(f"{name} length != num_states")
        if A:
            if not (0 <= self.arc_from.min() and self.arc_from.max() < S):
                raise TableFormatError("arc_from out of range")
            if not (0 <= self.arc_to.min() and self.arc_to.max() < S):
                raise TableFormatError("arc_to out of range")
            if not (0 <= self.arc_token.min() and self.arc_token.max() < V):
                raise TableFormatError("arc_token out of range")
            key = self.arc_from.astype(np.int64) * V + self.arc_token
            if not (np.diff(key) > 0).all():
                raise TableFormatError("arcs not strictly sorted by (from_state, token)")
        if not (0 <= self.backoff_to.min() and self.backoff_to.max() < S):
            raise TableFormatError("backoff_to out of range")
        lo = self.state_start.astype(np.int64)
        hi = self.state_end.astype(np.int64)
        bad = np.flatnonzero((lo < 0) | (lo > hi) | (hi > A))
        if bad.size:
            s = int(bad[0])
            raise TableFormatError(f"state {s}: bad arc range [{int(lo[s])}, {int(hi[s])})")
        counts = hi - lo
        if int(counts.sum()) > A:
            # overlapping ranges: some state covers a foreign arc; find the
            # first one as the reference's per-state loop does (table.py:113-117)
            # without materialising every range (S x A for a hostile file)
            for s in range(S):
                if counts[s] and not (self.arc_from[lo[s]:hi[s]] == s).all():
                    raise TableFormatError(f"state {s}: arc range covers foreign arcs")
            raise TableFormatError("arc ranges do not cover the arc array")
        if A and counts.sum():
            owner = np.repeat(np.arange(S), counts)
            ends = np.cumsum(counts)
            flat = np.arange(int(ends[-1]), dtype=np.int64) + np.repeat(lo - (ends - counts), counts)
            if (flat >= A).any():
                raise TableFormatError("arc ranges do not cover the arc array")
            mism = np.flatnonzero(self.arc_from[flat] != owner)
            if mism.size:
                raise TableFormatError(f"state {int(owner[mism[0]])}: arc range covers foreign arcs")
        if int(hi.sum() - lo.sum()) != A:
            raise TableFormatError("arc ranges do not cover the arc array")
        if int(self.backoff_to[0]) != 0 or float(self.backoff_weight[0]) != 0.0:
            raise TableFormatError("root backoff must be (0, 0)")
        fin = self.is_final.astype(bool)
        if fin.any() and not (self.backoff_weight[fin] == 0.0).all():
            raise TableFormatError("final states must have zero backoff weight")
        nonfinal = ~fin
        nonfinal[0] = False
        if nonfinal.any() and not (self.backoff_weight[nonfinal] <= 0.0).all():
            raise TableFormatError("non-final backoff weights must be <= 0")
        if not np.isfinite(self.arc_weight).all() or not np.isfinite(self.backoff_weight).all():
            raise TableFormatError("non-finite weight")

    # -- device copy ------------------------------------------------------
    def device_table(self, device: int | None = None) -> _DeviceTable:
        """The table's resident copy on `device` (default: current CUDA device)."""
        import torch

        _lib.require_cuda()
        dev = torch.cuda.current_device() if device is None else int(device)
        d = self._dev.get(dev)
        if d is None:
            with self._dev_lock:
                d = self._dev.get(dev)
                if d is None:
                    d = _DeviceTable(self, dev)
                    self._dev[dev] = d
        return d

    def __getstate__(self):
        st = self.__dict__.copy()
        st["_dev"] = {}
        st.pop("_dev_lock", None)
        return st

    def __setstate__(self, st):
        self.__dict__.update(st)
        self._dev = {}
        self._dev_lock = threading.Lock()


class DeviceTable:
    """A boosting table that lives only on one device: GPB1 bytes parsed,
    validated and laid out by the native loader (pgpb_table_load_gpb1), with
    no host ArcTable.  Accepted wherever the API takes a table for device
    work (get_scores_batch / advance, the greedy and beam decoders)."""

    def __init__(self, dt: _DeviceTable):
        info = dt.info()
        self._dt = dt
        self.num_states = int(info.num_states)
        self.vocab_size = int(info.vocab_size)
        self.num_arcs = int(info.num_arcs)
        self.unk_score = float(info.unk_score)
        self.device = dt.device

    def device_table(self, device: int | None = None) -> _DeviceTable:
        if device is not None and int(device) != self.device:
            raise ValueError(f"table resides on cuda:{self.device}, not cuda:{device}")
        return self._dt


def load_table_device(source, device: int | None = None) -> DeviceTable:
    """GPB1 file path (or bytes) straight to a device table (table.py:267-310
    semantics: TableFormatError on a malformed table)."""
    import torch

    _lib.require_cuda()
    dev = torch.cuda.current_device() if device is None else int(device)
    h = _lib.c_void_p()
    if isinstance(source, (bytes, bytearray, memoryview)):
        buf = np.frombuffer(bytes(source), dtype=np.uint8)
        rc = _lib.LIB.pgpb_table_load_gpb1(_lib.ptr(buf) if buf.size else None, buf.size, dev, _lib.ctypes.byref(h))
    else:
        rc = _lib.LIB.pgpb_table_load_gpb1_file(str(Path(source)).encode(), dev, _lib.ctypes.byref(h))
    if rc == _lib.PGPB_EFORMAT:
        raise TableFormatError(_lib.last_error())
    _lib.check(rc, "pgpb_table_load_gpb1")
    return DeviceTable(_DeviceTable._from_handle(h.value, dev))


@dataclass(frozen=True)
class ScoreQueryResult:
    """(B, V) boosting scores and next states (table.py:130-135)."""

    scores: object
    next_states: object


def compile_arc_table(tree: PrefixTree, unk_score: float = 0.0) -> ArcTable:
    """Flatten a fail-linked trie into an ArcTable (table.py:138-187)."""
    if not tree.has_fail_links:
        raise ValueError("tree has no fail links; run compute_fail_links first")
    S = tree.num_nodes
    A = S - 1
    arc_from = np.empty(A, np.int32)
    arc_token = np.empty(A, np.int32)
    arc_to = np.empty(A, np.int32)
    arc_weight = np.empty(A, np.float32)
    state_start = np.empty(S, np.int32)
    state_end = np.empty(S, np.int32)
    backoff_to = np.empty(S, np.int32)
    backoff_weight = np.empty(S, np.float32)
    final_score = np.empty(S, np.float32)
    fin = np.ascontiguousarray(tree.is_final, dtype=np.uint8)
    p = _lib.ptr
    _lib.check(_lib.LIB.pgpb_trie_compile(
        S, p(tree.parent), p(tree.in_token), p(fin), p(tree.arc_scores), p(tree.acc_scores),
        p(tree.fail), p(arc_from), p(arc_token), p(arc_to), p(arc_weight), p(state_start),
        p(state_end), p(backoff_to), p(backoff_weight), p(final_score),
    ), "pgpb_trie_compile")
    table = ArcTable(
        num_states=S, vocab_size=tree.vocab_size, arc_from=arc_from, arc_token=arc_token,
        arc_to=arc_to, arc_weight=arc_weight, state_start=state_start, state_end=state_end,
        backoff_to=backoff_to, backoff_weight=backoff_weight, is_final=tree.is_final.astype(bool),
        final_score=final_score, unk_score=float(unk_score),
    )
    table.validate()
    return table


def _is_tensor(x) -> bool:
    return type(x).__module__.startswith("torch") and hasattr(x, "is_cuda")


def get_scores_batch(table: ArcTable, states, *, check: bool = True, out=None) -> ScoreQueryResult:
    """Scores and next states of every token for each input state.

    numpy / list input: the reference's contract (table.py:190-214) — int32
    states, IndexError on out-of-range ids, fresh numpy (B, V) outputs; runs
    through the C-ABI host entry point (H2D, advance kernel, D2H).
    CUDA tensor input: device (B, V) float32 / int32 tensors, stream-ordered on
    torch's current stream (no sync unless `check` range-validates states).
    `out=(scores, next)` reuses caller-owned device buffers.
    """
    if _is_tensor(states):
        return _advance_device(table, states, check=check, out=out)
    st = np.ascontiguousarray(np.asarray(states, dtype=np.int32).reshape(-1))
    if st.size and (st.min() < 0 or st.max() >= table.num_states):
        raise IndexError(f"state id out of range [0, {table.num_states})")
    B, V = st.shape[0], table.vocab_size
    scores, nxt = _host_out(B, V)
    if B:
        dev = table.device_table()
        _lib.check(_lib.LIB.pgpb_advance_host(
            dev.handle, _lib.ptr(st), B, _lib.ptr(scores), _lib.ptr(nxt), _lib.stream_ptr(),
        ), "pgpb_advance_host")
    return ScoreQueryResult(scores=scores, next_states=nxt)


def _host_out(B: int, V: int):
    """Fresh (B, V) float32 / int32 host outputs in page-locked memory, so the
    device-to-host copy of the result runs at full link speed.  The arrays
    are ordinary numpy arrays (they keep their pinned torch storage alive)."""
    import torch

    if B * V == 0:
        return np.empty((B, V), np.float32), np.empty((B, V), np.int32)
    s = torch.empty((B, V), dtype=torch.float32, pin_memory=True)
    n = torch.empty((B, V), dtype=torch.int32, pin_memory=True)
    return s.numpy(), n.numpy()


def _advance_device(table: ArcTable, states, *, check: bool, out, chain: bool = False) -> ScoreQueryResult:
    import torch

    if not states.is_cuda:
        raise ValueError("states tensor must live on a CUDA device (or pass numpy)")
    st = states.reshape(-1)
    if st.dtype != torch.int32:
        st = st.to(torch.int32)
    st = st.contiguous()
    B, V = st.shape[0], table.vocab_size
    if check and B:
        lo, hi = torch.aminmax(st)
        if int(lo) < 0 or int(hi) >= table.num_states:
            raise IndexError(f"state id out of range [0, {table.num_states})")
    if out is None:
        scores = torch.empty((B, V), dtype=torch.float32, device=st.device)
        nxt = torch.empty((B, V), dtype=torch.int32, device=st.device)
    else:
        scores, nxt = out
        if tuple(scores.shape) != (B, V) or tuple(nxt.shape) != (B, V):
            raise ValueError("out buffers must be (B, V)")
    if B:
        dev = table.device_table(st.device.index)
        fn = _lib.LIB.pgpb_advance_chain if chain else _lib.LIB.pgpb_advance
        _lib.check(fn(dev.handle, st.data_ptr(), B, scores.data_ptr(), nxt.data_ptr(),
                      _lib.stream_ptr()), "pgpb_advance")
    return ScoreQueryResult(scores=scores, next_states=nxt)


def advance(table: ArcTable, states, **kw) -> ScoreQueryResult:
    """north_star name for get_scores_batch: advance(states) -> (scores, next_states)."""
    return get_scores_batch(table, states, **kw)


@dataclass(frozen=True)
class AdvanceStepsResult:
    """R chained advances: scores / next_states (R, B, V), the state each step
    queried (trace, (R, B)) and the state after the last step (final, (B,))."""

    scores: object
    next_states: object
    trace: object
    final_states: object


def advance_steps(table, states, tokens, *, parts: int = 0, out=None, check: bool = True) -> AdvanceStepsResult:
    """R chained advances in one launch (pgpb_advance_steps, BASELINE config 5):
    step k = get_scores_batch of the step's states (table.py:190-214);
    s_{k+1}[b] = next_k[b, tokens[k, b]] (the reference's next-state lookup,
    decoding.py:379-383).  `states` int32 (B,) and `tokens` int32 (R, B) CUDA
    tensors; outputs are device tensors on torch's current stream."""
    import torch

    if not (_is_tensor(states) and states.is_cuda and _is_tensor(tokens) and tokens.is_cuda):
        raise ValueError("advance_steps takes CUDA tensors (states (B,), tokens (R, B))")
    st = states.reshape(-1).to(torch.int32).contiguous()
    tk = tokens.to(torch.int32).contiguous()
    B, V = st.shape[0], table.vocab_size
    if tk.dim() != 2 or tk.shape[1] != B:
        raise ValueError("tokens must be (R, B)")
    R = tk.shape[0]
    if check and B:
        lo, hi = torch.aminmax(st)
        if int(lo) < 0 or int(hi) >= table.num_states:
            raise IndexError(f"state id out of range [0, {table.num_states})")
        if R:
            lo, hi = torch.aminmax(tk)
            if int(lo) < 0 or int(hi) >= V:
                raise IndexError(f"token id out of range [0, {V})")
    dev_ = st.device
    if out is None:
        scores = torch.empty((R, B, V), dtype=torch.float32, device=dev_)
        nxt = torch.empty((R, B, V), dtype=torch.int32, device=dev_)
    else:
        scores, nxt = out
        if tuple(scores.shape) != (R, B, V) or tuple(nxt.shape) != (R, B, V):
            raise ValueError("out buffers must be (R, B, V)")
    trace = torch.empty((R, B), dtype=torch.int32, device=dev_)
    final = st.clone()
    if B and R:
        dt = table.device_table(dev_.index)
        _lib.check(_lib.LIB.pgpb_advance_steps(dt.handle, st.data_ptr(), tk.data_ptr(), R, B, scores.data_ptr(),
                                               nxt.data_ptr(), trace.data_ptr(), final.data_ptr(), int(parts),
                                               _lib.stream_ptr()), "pgpb_advance_steps")
    return AdvanceStepsResult(scores=scores, next_states=nxt, trace=trace, final_states=final)


def naive_score(tree: PrefixTree, state: int, token: int, unk_score: float = 0.0) -> tuple[float, int]:
    """Single-cell resolution on the trie itself (table.py:217-247), fp32 like compile."""
    if not 0 <= state < tree.num_nodes:
        raise IndexError(f"state id {state} out of range")
    if not 0 <= token < tree.vocab_size:
        raise IndexError(f"token id {token} out of range")
    if not tree.has_fail_links:
        raise ValueError("tree has no fail links; run compute_fail_links first")
    f32 = np.float32
    acc = f32(0.0)
    cur = int(state)
    while True:
        hit = tree.lookup(cur, token)
        if hit >= 0:
            return float(acc + f32(tree.arc_scores[hit])), hit
        if cur == 0:
            return float(acc + f32(unk_score)), 0
        nxt = int(tree.fail[cur])
        bw = f32(0.0) if tree.is_final[cur] else f32(tree.acc_scores[nxt] - tree.acc_scores[cur])
        acc = f32(acc + bw)
        cur = nxt


def save_table(table: ArcTable, path) -> None:
    """GPB1 little-endian serialisation (table.py:16-29, :250-266)."""
    table.validate()
    blob = b"".join([
        _HEADER.pack(MAGIC, VERSION, table.num_states, table.vocab_size, table.num_arcs, table.unk_score),
        *(np.ascontiguousarray(getattr(table, n), dtype=dt).tobytes() for n, dt in _GPB1_FIELDS),
    ])
    Path(path).write_bytes(blob)


_GPB1_FIELDS = (
    ("arc_from", "<i4"), ("arc_token", "<i4"), ("arc_to", "<i4"), ("arc_weight", "<f4"),
    ("state_start", "<i4"), ("state_end", "<i4"), ("backoff_to", "<i4"), ("backoff_weight", "<f4"),
    ("is_final", "<u1"), ("final_score", "<f4"),
)


def load_table(path) -> ArcTable:
    """Read and validate a GPB1 file (table.py:269-310)."""
    blob = Path(path).read_bytes()
    if len(blob) < _HEADER.size:
        raise TableFormatError(f"{path}: truncated header")
    magic, version, S, V, A, unk = _HEADER.unpack_from(blob, 0)
    if magic != MAGIC:
        raise TableFormatError(f"{path}: bad magic {magic!r}")
    if version != VERSION:
        raise TableFormatError(f"{path}: unsupported version {version}")
    expected = _HEADER.size + 16 * A + 21 * S
    if len(blob) != expected:
        raise TableFormatError(f"{path}: expected {expected} bytes, found {len(blob)}")
    arrays = {}
    off = _HEADER.size
    for name, dt in _GPB1_FIELDS:
        count = A if name.startswith("arc_") else S
        a = np.frombuffer(blob, dtype=dt, count=count, offset=off).copy()
        off += a.nbytes
        arrays[name] = a
    arrays["is_final"] = arrays["is_final"].astype(bool)
    table = ArcTable(num_states=S, vocab_size=V, unk_score=float(unk), **arrays)
    try:
        table.validate()
    except TableFormatError as exc:
        raise TableFormatError(f"{path}: corrupt table: {exc}") from None
    return table


def state_strings(table: ArcTable, vocab: Vocabulary | None = None) -> list[str]:
    """Token-path label of every state, recovered from tree arcs (table.py:313-333)."""
    S = table.num_states
    par = np.full(S, -1, np.int64)
    tok = np.full(S, -1, np.int64)
    to = table.arc_to.astype(np.int64)
    first = np.ones(to.shape[0], bool)
    _, idx = np.unique(to, return_index=True)
    first[:] = False
    first[idx] = True
    sel = first & (to != 0)
    par[to[sel]] = table.arc_from[sel]
    tok[to[sel]] = table.arc_token[sel]
    labels = [""] * S
    for s in range(1, S):
        ids = []
        cur = s
        while cur != 0:
            ids.append(int(tok[cur]))
            cur = int(par[cur])
        ids.reverse()
        labels[s] = "".join(vocab.tokens[i] for i in ids) if vocab is not None else ",".join(map(str, ids))
    return labels
