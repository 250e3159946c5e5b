"""Shallow-fusion decoders on the GPU: greedy / beam CTC, transducer, AED.

API mirror of the reference's `phraseboost.decoding`
(/root/reference/pkg/src/phraseboost/decoding.py).  Ranking is
am + lam * boost everywhere; blank / CTC repeats never touch the tree; with
lam == 0, boosting disabled or no table the tree is skipped entirely
(decoding.py:103-104), so baselines are identical whichever switch is off.

What runs where:
  * ctc_greedy_boosted / ctc_greedy_boosted_batch -> fused batched greedy
    kernel (pgpb_ctc_greedy): argmax, blank/repeat pass-through and the
    fp64 boosted rerank, the [B,V] score matrix never written.
  * transducer_greedy_boosted -> pgpb_greedy_step per symbol (the batched,
    CUDA-graph label-looping variant lives in rnnt.py).
  * ctc_beam_boosted / transducer_beam_boosted / aed_beam_boosted -> the
    fused expansion + top-k kernel (pgpb_beam_topk) for every V-wide step;
    only the O(beam) hypothesis bookkeeping (prefix merges, eos handling)
    stays on the host.  Any beam width: the kernel's top-k runs in exact
    passes of 32 winners.
There is no CPU scoring path: the advance/rerank always runs on the GPU.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np

from . import _lib
from .acoustic import FLAVOR_AED, FLAVOR_TRANSDUCER, EmissionMatrix, StepModel
from .context import Vocabulary, detokenize
from .table import ArcTable, get_scores_batch

NEG_INF = float("-inf")
DEFAULT_BEAM_CTC = 8
DEFAULT_BEAM_TRANSDUCER = 8
DEFAULT_BEAM_AED = 3


@dataclass(frozen=True)
class DecodeConfig:
    """decoding.py:44-60."""

    lam: float = 1.0
    beam_size: int = 8
    max_symbols_per_frame: int = 5
    eos_bump_enabled: bool = True
    boost_enabled: bool = True
    # Extension with no reference counterpart (parity unpinned, off by
    # default): when a beam hypothesis is finalised (last frame for CTC /
    # transducer beams, eos for AED) its boost takes back the unfinished
    # phrase's credit, i.e. adds the state's backoff total.
    rollback: bool = False

    def __post_init__(self):
        if self.lam < 0:
            raise ValueError(f"lam must be >= 0, got {self.lam}")
        if self.beam_size < 1:
            raise ValueError(f"beam_size must be >= 1, got {self.beam_size}")
        if self.max_symbols_per_frame < 1:
            raise ValueError(f"max_symbols_per_frame must be >= 1, got {self.max_symbols_per_frame}")


@dataclass(frozen=True)
class TraceStep:
    token: int
    boost: float
    state: int


@dataclass
class DecodeResult:
    tokens: list[int]
    text: str
    am_score: float
    boost_score: float
    trace: list[TraceStep] | None = None


@dataclass
class Hypothesis:
    tokens: tuple[int, ...]
    am_score: float
    boost_score: float
    tree_state: int
    last_token: int | None = None
    ended: bool = False
    trace: tuple[TraceStep, ...] = ()


def _logaddexp(a: float, b: float) -> float:
    """decoding.py:94-100 (host fp64, same libm as the reference)."""
    if a == NEG_INF:
        return b
    if b == NEG_INF:
        return a
    hi = a if a > b else b
    return hi + math.log1p(math.exp(-abs(a - b)))


def _boost_active(table: ArcTable | None, cfg: DecodeConfig) -> bool:
    return table is not None and cfg.boost_enabled and cfg.lam != 0.0


def _text(tokens, vocab: Vocabulary | None) -> str:
    return "" if vocab is None else detokenize(tokens, vocab)


def _check_ctc_inputs(em: EmissionMatrix, table: ArcTable | None) -> None:
    if em.blank_id is None:
        raise ValueError("CTC decoding needs em.blank_id")
    if table is not None and em.vocab_size != table.vocab_size:
        raise ValueError(f"emission vocab size {em.vocab_size} != table vocab size {table.vocab_size}")


def _check_step_inputs(step: StepModel, flavor: str, table: ArcTable | None) -> None:
    if step.flavor != flavor:
        raise ValueError(f"step model flavor {step.flavor!r} != {flavor!r}")
    if table is not None and step.vocab_size != table.vocab_size:
        raise ValueError(f"step model vocab size {step.vocab_size} != table vocab size {table.vocab_size}")


def _torch():
    import torch

    _lib.require_cuda()
    return torch


def _handle(table: ArcTable | None, use_boost: bool, device=None):
    return table.device_table(device).handle if (use_boost and table is not None) else None


def _rank_key(lam: float):
    return lambda h: (-(h.am_score + lam * h.boost_score), -h.am_score, h.tokens)


def _keep_better(pool: dict, key, cand: Hypothesis, lam: float) -> None:
    """decoding.py:396-404."""
    old = pool.get(key)
    if old is None or (cand.am_score + lam * cand.boost_score, cand.am_score) > (
        old.am_score + lam * old.boost_score, old.am_score
    ):
        pool[key] = cand


def _results(beam, lam, beam_size, vocab, want_trace):
    return [
        DecodeResult(list(h.tokens), _text(h.tokens, vocab), h.am_score, h.boost_score,
                     list(h.trace) if want_trace else None)
        for h in sorted(beam, key=_rank_key(lam))[:beam_size]
    ]


# ---------------------------------------------------------------------------
# Greedy CTC


def ctc_greedy_boosted(em: EmissionMatrix, table: ArcTable | None = None, cfg: DecodeConfig | None = None, *,
                       vocab: Vocabulary | None = None, want_trace: bool = False) -> DecodeResult:
    """Two-stage greedy CTC (decoding.py:156-229) through the C-ABI host entry."""
    cfg = cfg or DecodeConfig()
    _check_ctc_inputs(em, table)
    use = _boost_active(table, cfg)
    _lib.require_cuda()
    T, V = em.logprobs.shape
    tok = np.empty(T, np.int32)
    dl = np.empty(T, np.float64)
    st = np.empty(T, np.int32)
    n = _lib.c_int64()
    am = _lib.c_double()
    bo = _lib.c_double()
    _lib.check(_lib.LIB.pgpb_ctc_greedy_host(
        _handle(table, use), _lib.ptr(em.logprobs), T, V, int(em.blank_id), float(cfg.lam), int(use),
        _lib.ptr(tok), _lib.ptr(dl), _lib.ptr(st), _lib.ctypes.byref(n), _lib.ctypes.byref(am),
        _lib.ctypes.byref(bo), _lib.stream_ptr(),
    ), "pgpb_ctc_greedy_host")
    k = n.value
    tokens = [int(x) for x in tok[:k]]
    trace = [TraceStep(int(a), float(b), int(c)) for a, b, c in zip(tok[:k], dl[:k], st[:k])] if want_trace else None
    return DecodeResult(tokens, _text(tokens, vocab), float(am.value), float(bo.value), trace)


@dataclass
class GreedyBatchOutput:
    """Device outputs of ctc_greedy_device (all on the logprobs' device)."""

    tokens: object  # int32 [B, T]
    deltas: object  # float64 [B, T]
    states: object  # int32 [B, T]
    num_out: object  # int32 [B]
    am: object  # float64 [B]
    boost: object  # float64 [B]


def ctc_greedy_device(logprobs, lengths, table: ArcTable | None, cfg: DecodeConfig, blank_id: int, *,
                      out: GreedyBatchOutput | None = None, stream=None) -> GreedyBatchOutput:
    """Batched fused greedy CTC on device tensors, no host synchronisation.

    logprobs: float32 CUDA tensor [B, T, V]; lengths: int32 CUDA tensor [B] or None.
    Lengths are not validated here (no host synchronisation); the kernels
    clamp them to [0, T], so a bad length never addresses another row.
    """
    torch = _torch()
    if logprobs.dim() != 3 or logprobs.dtype != torch.float32 or not logprobs.is_cuda:
        raise ValueError("logprobs must be a float32 CUDA tensor [B, T, V]")
    lp = logprobs.contiguous()
    B, T, V = lp.shape
    if table is not None and V != table.vocab_size:
        raise ValueError(f"emission vocab size {V} != table vocab size {table.vocab_size}")
    use = _boost_active(table, cfg)
    dev = lp.device
    if out is None:
        out = GreedyBatchOutput(
            torch.empty((B, T), dtype=torch.int32, device=dev), torch.empty((B, T), dtype=torch.float64, device=dev),
            torch.empty((B, T), dtype=torch.int32, device=dev), torch.empty(B, dtype=torch.int32, device=dev),
            torch.empty(B, dtype=torch.float64, device=dev), torch.empty(B, dtype=torch.float64, device=dev),
        )
    if lengths is not None:
        lengths = lengths.to(device=dev, dtype=torch.int32).contiguous()
    _lib.check(_lib.LIB.pgpb_ctc_greedy(
        _handle(table, use, dev.index), lp.data_ptr(), B, T, V,
        None if lengths is None else lengths.data_ptr(), int(blank_id), float(cfg.lam), int(use),
        out.tokens.data_ptr(), out.deltas.data_ptr(), out.states.data_ptr(), out.num_out.data_ptr(),
        out.am.data_ptr(), out.boost.data_ptr(), _lib.stream_ptr(stream),
    ), "pgpb_ctc_greedy")
    return out


def ctc_greedy_boosted_batch(logprobs, lengths=None, table: ArcTable | None = None, cfg: DecodeConfig | None = None,
                             *, blank_id: int, vocab: Vocabulary | None = None,
                             want_trace: bool = False) -> list[DecodeResult]:
    """Greedy CTC over a batch; each result equals the per-utterance call.

    logprobs: [B, T, V] float32 (numpy or CUDA tensor); lengths: [B] frames.
    """
    torch = _torch()
    cfg = cfg or DecodeConfig()
    lp = logprobs if isinstance(logprobs, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(logprobs, np.float32))
    lp = lp.to(device="cuda", dtype=torch.float32)
    ln = None if lengths is None else torch.as_tensor(np.asarray(lengths) if not isinstance(lengths, torch.Tensor) else lengths)
    if ln is not None:
        if tuple(ln.shape) != (lp.shape[0],):
            raise ValueError(f"lengths must have shape ({lp.shape[0]},), got {tuple(ln.shape)}")
        lo, hi = (int(x) for x in torch.aminmax(ln.to(torch.int64))) if ln.numel() else (0, 0)
        if lo < 0 or hi > lp.shape[1]:
            raise ValueError(f"lengths must lie in [0, {lp.shape[1]}], got [{lo}, {hi}]")
    B, T = lp.shape[0], lp.shape[1]
    z = lambda *shape, dt: torch.zeros(shape, dtype=dt, device=lp.device)  # noqa: E731
    # zero-filled: the whole [B, T] arrays are copied back, slots past num_out included
    o = ctc_greedy_device(lp, ln, table, cfg, blank_id, out=GreedyBatchOutput(
        z(B, T, dt=torch.int32), z(B, T, dt=torch.float64), z(B, T, dt=torch.int32), z(B, dt=torch.int32),
        z(B, dt=torch.float64), z(B, dt=torch.float64)))
    n = o.num_out.cpu().numpy()
    tok, dl, st = o.tokens.cpu().numpy(), o.deltas.cpu().numpy(), o.states.cpu().numpy()
    am, bo = o.am.cpu().numpy(), o.boost.cpu().numpy()
    res = []
    for b in range(lp.shape[0]):
        k = int(n[b])
        tokens = [int(x) for x in tok[b, :k]]
        trace = [TraceStep(int(a), float(c), int(s)) for a, c, s in zip(tok[b, :k], dl[b, :k], st[b, :k])] if want_trace else None
        res.append(DecodeResult(tokens, _text(tokens, vocab), float(am[b]), float(bo[b]), trace))
    return res


# ---------------------------------------------------------------------------
# Greedy transducer (host StepModel)


class _StepRunner:
    """Device staging for pgpb_greedy_step on `rows` host rows."""

    def __init__(self, table, use, V, blank, lam, rows=1):
        torch = _torch()
        self.torch = torch
        self.h = _handle(table, use)
        self.use, self.V, self.blank, self.lam = use, V, blank, lam
        d = "cuda"
        self.lp_host = torch.empty((rows, V), dtype=torch.float32, pin_memory=True)
        self.lp = torch.empty((rows, V), dtype=torch.float32, device=d)
        self.states = torch.zeros(rows, dtype=torch.int32, device=d)
        self.chosen = torch.empty(rows, dtype=torch.int32, device=d)
        self.lpc = torch.empty(rows, dtype=torch.float32, device=d)
        self.delta = torch.empty(rows, dtype=torch.float64, device=d)
        self.nxt = torch.empty(rows, dtype=torch.int32, device=d)
        self.blk = torch.empty(rows, dtype=torch.uint8, device=d)

    def run(self, row: np.ndarray, state: int):
        self.lp_host[0].copy_(self.torch.from_numpy(np.ascontiguousarray(row, np.float32)))
        self.lp.copy_(self.lp_host, non_blocking=True)
        self.states.fill_(int(state))
        _lib.check(_lib.LIB.pgpb_greedy_step(
            self.h, self.lp.data_ptr(), self.V, 1, self.V, self.states.data_ptr(), None, int(self.blank),
            float(self.lam), int(self.use), self.chosen.data_ptr(), self.lpc.data_ptr(), self.delta.data_ptr(),
            self.nxt.data_ptr(), self.blk.data_ptr(), _lib.stream_ptr(),
        ), "pgpb_greedy_step")
        packed = self.torch.stack([self.chosen.double(), self.nxt.double(), self.blk.double(), self.delta]).cpu()
        c, nx, bl, d = packed[:, 0].tolist()
        return int(c), bool(bl), d, int(nx)


def transducer_greedy_boosted(step: StepModel, num_frames: int, blank_id: int, table: ArcTable | None = None,
                              cfg: DecodeConfig | None = None, *, vocab: Vocabulary | None = None,
                              want_trace: bool = False) -> DecodeResult:
    """Frame-synchronous greedy transducer with a per-frame symbol cap (decoding.py:350-393)."""
    cfg = cfg or DecodeConfig()
    _check_step_inputs(step, FLAVOR_TRANSDUCER, table)
    use = _boost_active(table, cfg)
    runner = _StepRunner(table, use, step.vocab_size, blank_id, cfg.lam)
    tokens: list[int] = []
    trace: list[TraceStep] = []
    am = boost = 0.0
    state = 0
    last: int | None = None
    for t in range(num_frames):
        for _ in range(cfg.max_symbols_per_frame):
            row = step.logprobs(last, t)
            chosen, is_blank, delta, nxt = runner.run(row, state)
            if is_blank:
                am += float(row[blank_id])
                break
            tokens.append(chosen)
            if want_trace:
                trace.append(TraceStep(chosen, delta, nxt))
            am += float(row[chosen])
            boost += delta
            state = nxt
            last = chosen
    return DecodeResult(tokens, _text(tokens, vocab), am, boost, trace if want_trace else None)


# ---------------------------------------------------------------------------
# Fused beam expansion (pgpb_beam_topk)


class _TopK:
    """pgpb_beam_topk for a single group of hypotheses.

    The device orders candidates by (combined, am, hypothesis, token); the
    reference ranks equal (combined, am) by token tuple instead
    (decoding.py:323-327, :407-411).  So that exact ties at the cut cannot
    change which candidates survive, the result is extended past k by every
    candidate tied with the k-th (fetched on demand: normally one extra
    candidate shows there is no tie), and the callers re-rank with the
    reference's full key before truncating."""

    def __init__(self, table, use, V, lam):
        self.torch = _torch()
        self.h = _handle(table, use)
        self.use, self.V, self.lam = use, V, float(lam)

    def __call__(self, rows_dev, ld, states, am, boost, exclude, k, alt_token=None, alt_am=None,
                 valid=None, skip_neg_inf=False):
        H = len(am)
        k = min(int(k), H * self.V)  # never more winners than candidates
        if k <= 0:
            return []
        lam = self.lam

        def tie(a, b):
            return a[2] == b[2] and a[2] + lam * a[3] == b[2] + lam * b[3]

        kr = min(k + 1, H * self.V)
        while True:
            out = self._run(rows_dev, ld, states, am, boost, exclude, kr, alt_token, alt_am, valid, skip_neg_inf)
            if len(out) <= k or not tie(out[k - 1], out[-1]) or len(out) < kr or kr == H * self.V:
                break
            kr = min(2 * kr, H * self.V)  # the tie group may run past what was fetched
        n = min(k, len(out))
        while n < len(out) and tie(out[k - 1], out[n]):
            n += 1
        return out[:n]

    def _run(self, rows_dev, ld, states, am, boost, exclude, k, alt_token, alt_am, valid, skip_neg_inf):
        torch = self.torch
        H = len(am)
        dev = rows_dev.device

        def t(x, dt):
            return None if x is None else torch.as_tensor(np.asarray(x), dtype=dt).to(dev, non_blocking=True)

        st = t(states, torch.int32)
        a = t(am, torch.float64)
        b = t(boost, torch.float64)
        ex = t(exclude, torch.int32)
        at = t(alt_token, torch.int32)
        aa = t(alt_am, torch.float64)
        va = t(valid, torch.uint8)
        o_h = torch.empty(k, dtype=torch.int32, device=dev)
        o_t = torch.empty(k, dtype=torch.int32, device=dev)
        o_am = torch.empty(k, dtype=torch.float64, device=dev)
        o_b = torch.empty(k, dtype=torch.float64, device=dev)
        o_n = torch.empty(k, dtype=torch.int32, device=dev)
        o_d = torch.empty(k, dtype=torch.float32, device=dev)
        p = lambda x: None if x is None else x.data_ptr()  # noqa: E731
        _lib.check(_lib.LIB.pgpb_beam_topk(
            self.h, rows_dev.data_ptr(), ld, H, self.V, H, k, p(st), p(a), p(b), p(ex), p(at), p(aa), p(va),
            self.lam, int(self.use), int(skip_neg_inf), p(o_h), p(o_t), p(o_am), p(o_b), p(o_n), p(o_d),
            _lib.stream_ptr(),
        ), "pgpb_beam_topk")
        ints = torch.stack([o_h, o_t, o_n]).cpu().numpy()
        flts = torch.stack([o_am, o_b, o_d.double()]).cpu().numpy()
        out = []
        for j in range(k):
            if ints[0, j] < 0:
                break
            out.append((int(ints[0, j]), int(ints[1, j]), float(flts[0, j]), float(flts[1, j]),
                        int(ints[2, j]), float(flts[2, j])))
        return out


def _backoff_totals(table, use: bool, cfg: DecodeConfig):
    """Per-state backoff totals (host copy) for the rollback extension, or None."""
    if not (use and cfg.rollback):
        return None
    return table.device_table().backoff_total().cpu().numpy()


def _rows_to_device(rows: np.ndarray):
    torch = _torch()
    return torch.from_numpy(np.ascontiguousarray(rows, np.float32)).to("cuda", non_blocking=True)


# ---------------------------------------------------------------------------
# CTC prefix beam


class _Prefix:
    __slots__ = ("pb", "pnb", "state", "boost", "trace")

    def __init__(self, pb, pnb, state, boost, trace):
        self.pb, self.pnb, self.state, self.boost, self.trace = pb, pnb, state, boost, trace

    @property
    def am(self) -> float:
        return _logaddexp(self.pb, self.pnb)


def _prefix_rank(lam):
    return lambda kv: (-(kv[1].am + lam * kv[1].boost), -kv[1].am, kv[0])


def ctc_beam_boosted(em: EmissionMatrix, table: ArcTable | None = None, cfg: DecodeConfig | None = None, *,
                     vocab: Vocabulary | None = None, want_trace: bool = False):
    """CTC prefix beam search (decoding.py:247-343, R8).

    Per frame the V-wide expansion of every live prefix and its top-k run in
    one fused kernel; the host adds the O(beam) carries (blank / repeat
    mass and extensions that land on an existing prefix) with the
    reference's fp64 log-add-exp, so scores are bit-identical.
    """
    cfg = cfg or DecodeConfig()
    _check_ctc_inputs(em, table)
    use = _boost_active(table, cfg)
    blank, lam, beam = em.blank_id, cfg.lam, cfg.beam_size
    lp = em.logprobs
    lp_dev = _rows_to_device(lp)
    V = em.vocab_size
    topk = _TopK(table, use, V, lam)
    entries: dict[tuple, _Prefix] = {(): _Prefix(0.0, NEG_INF, 0, 0.0, ())}
    rank = _prefix_rank(lam)
    for t in range(em.num_frames):
        items = list(entries.items())
        idx = {p: i for i, (p, _) in enumerate(items)}
        tot = [_logaddexp(e.pb, e.pnb) for _, e in items]
        lastv = [p[-1] if p else -1 for p, _ in items]
        lb = float(lp[t, blank])
        new: dict[tuple, _Prefix] = {}
        # carries: blank / repeat mass on each live prefix, plus the extension
        # from its parent prefix when that parent is also live
        for j, (p, e) in enumerate(items):
            pnb = NEG_INF
            if p:
                i = idx.get(p[:-1])
                if i is not None:
                    v = p[-1]
                    contrib = (items[i][1].pb if v == lastv[i] else tot[i]) + float(lp[t, v])
                    if contrib != NEG_INF:
                        pnb = contrib
                pnb = _logaddexp(pnb, e.pnb + float(lp[t, p[-1]]))
            new[p] = _Prefix(tot[j] + lb, pnb, e.state, e.boost, e.trace)
        # extensions to new prefixes: fused kernel top-k
        k = beam + len(items)
        cands = topk(lp_dev[t], 0, [e.state for _, e in items], tot, [e.boost for _, e in items],
                     [blank] * len(items), k, alt_token=lastv, alt_am=[e.pb for _, e in items],
                     skip_neg_inf=True)
        for h, v, amv, bov, nxt, delta in cands:
            np_ = items[h][0] + (v,)
            if np_ in idx:
                continue  # already merged into the carry above
            d = delta if use else 0.0
            tr = items[h][1].trace + (TraceStep(v, d, nxt),) if want_trace else ()
            new[np_] = _Prefix(NEG_INF, amv, nxt, bov, tr)
        entries = dict(sorted(new.items(), key=rank)[:beam])
    bt = _backoff_totals(table, use, cfg)
    if bt is not None and em.num_frames > 0:
        for e in entries.values():
            e.boost = e.boost + float(bt[e.state])
    ranked = sorted(entries.items(), key=rank)[:beam]
    nbest = [DecodeResult(list(p), _text(p, vocab), e.am, e.boost, list(e.trace) if want_trace else None)
             for p, e in ranked]
    return nbest[0], nbest



# ---------------------------------------------------------------------------
# Transducer beam


def transducer_beam_boosted(step: StepModel, num_frames: int, blank_id: int, table: ArcTable | None = None,
                            cfg: DecodeConfig | None = None, *, vocab: Vocabulary | None = None,
                            want_trace: bool = False):
    """Frame-synchronous transducer beam search (decoding.py:428-495, R9).

    Each expansion wave is one fused kernel call: all non-blank expansions
    of the wave's hypotheses are scored and reduced to the top `beam`
    on the GPU (expansions of distinct token sequences never collide, so
    no merge is lost).  Blank extensions merge into `finished` on the host.
    """
    cfg = cfg or DecodeConfig()
    _check_step_inputs(step, FLAVOR_TRANSDUCER, table)
    use = _boost_active(table, cfg)
    lam, beam_size, cap, V = cfg.lam, cfg.beam_size, cfg.max_symbols_per_frame, step.vocab_size
    rank = _rank_key(lam)
    topk = _TopK(table, use, V, lam)
    bt = _backoff_totals(table, use, cfg)
    beam = [Hypothesis((), 0.0, 0.0, 0)]
    for t in range(num_frames):
        active: dict = {}
        for h in beam:
            _keep_better(active, (h.tokens, 0), h, lam)
        finished: dict = {}
        while active:
            waves = sorted(active.items(), key=lambda kv: rank(kv[1]))
            rows = np.stack([step.logprobs(h.last_token, t) for _, h in waves]).astype(np.float32)
            for i, ((_, k), h) in enumerate(waves):
                _keep_better(finished, h.tokens, replace(h, am_score=h.am_score + float(rows[i, blank_id])), lam)
            k_wave = waves[0][0][1]
            if k_wave >= cap:
                break
            hyps = [h for _, h in waves]
            cands = topk(_rows_to_device(rows), V, [h.tree_state for h in hyps], [h.am_score for h in hyps],
                         [h.boost_score for h in hyps], [blank_id] * len(hyps), beam_size)
            # the reference's prune order, token tuples breaking exact ties (decoding.py:490)
            cands = sorted(cands, key=lambda c: (-(c[2] + lam * c[3]), -c[2], hyps[c[0]].tokens + (c[1],)))
            nxt_active = {}
            for hi, v, amv, bov, nxt, delta in cands[:beam_size]:
                h = hyps[hi]
                d = delta if use else 0.0
                c = Hypothesis(h.tokens + (v,), amv, bov, nxt, v,
                               trace=h.trace + (TraceStep(v, d, nxt),) if want_trace else ())
                nxt_active[(c.tokens, k_wave + 1)] = c
            active = nxt_active
        if bt is not None and t == num_frames - 1:
            finished = {k: replace(h, boost_score=h.boost_score + float(bt[h.tree_state])) for k, h in finished.items()}
        beam = sorted(finished.values(), key=rank)[:beam_size]
    nbest = _results(beam, lam, beam_size, vocab, want_trace)
    return nbest[0], nbest



# ---------------------------------------------------------------------------
# AED beam


def aed_beam_boosted(step: StepModel, table: ArcTable | None = None, cfg: DecodeConfig | None = None, *,
                     max_len: int, vocab: Vocabulary | None = None, want_trace: bool = False):
    """Label-synchronous beam with the eos anti-suppression bump (decoding.py:502-587, R10).

    Non-eos expansions of all active hypotheses: one fused top-k kernel call
    per step.  The eos bump uses the per-state row maximum computed once per
    table on the GPU (pgpb_row_max).
    """
    cfg = cfg or DecodeConfig()
    _check_step_inputs(step, FLAVOR_AED, table)
    if step.eos_id is None:
        raise ValueError("AED decoding needs step.eos_id")
    if max_len < 1:
        raise ValueError(f"max_len must be >= 1, got {max_len}")
    use = _boost_active(table, cfg)
    lam, eos, V, beam_size = cfg.lam, step.eos_id, step.vocab_size, cfg.beam_size
    rank = _rank_key(lam)
    topk = _TopK(table, use, V, lam)
    row_max = final_bonus = None
    if use and cfg.eos_bump_enabled:  # device arrays: works for ArcTable and DeviceTable alike
        row_max = table.device_table().row_max().cpu().numpy()
        final_bonus = table.device_table().final_bonus().cpu().numpy()
    bt = _backoff_totals(table, use, cfg)
    beam = [Hypothesis((), 0.0, 0.0, 0)]
    while True:
        active = [h for h in beam if not h.ended and len(h.tokens) < max_len]
        if not active:
            break
        cands = [h for h in beam if h.ended or len(h.tokens) >= max_len]
        rows = np.stack([step.logprobs(h.tokens, len(h.tokens)) for h in active]).astype(np.float32)
        for i, h in enumerate(active):
            bump = 0.0
            if row_max is not None:
                best = float(row_max[h.tree_state])
                bump = best if best > 0.0 else 0.0
                bump += float(final_bonus[h.tree_state])  # 0 unless final (decoding.py:551-552)
            if bt is not None:
                bump += float(bt[h.tree_state])
            cands.append(Hypothesis(h.tokens, h.am_score + float(rows[i, eos]), h.boost_score + bump, h.tree_state,
                                    h.last_token, ended=True,
                                    trace=h.trace + (TraceStep(eos, bump, h.tree_state),) if want_trace else ()))
        ext = topk(_rows_to_device(rows), V, [h.tree_state for h in active], [h.am_score for h in active],
                   [h.boost_score for h in active], [eos] * len(active), beam_size)
        for hi, v, amv, bov, nxt, delta in ext:
            h = active[hi]
            d = delta if use else 0.0
            cands.append(Hypothesis(h.tokens + (v,), amv, bov, nxt, v,
                                    trace=h.trace + (TraceStep(v, d, nxt),) if want_trace else ()))
        beam = sorted(cands, key=rank)[:beam_size]
    nbest = _results(beam, lam, beam_size, vocab, want_trace)
    return nbest[0], nbest


