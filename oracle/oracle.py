"""ORACLE — TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference's hot path, used by tests/, by
__graft_entry__.smoke() and by bench.py's CPU-baseline legs — never by the
product (paper_2508_07014_b200/ does not import this package).

Contents (each follows the cited reference file:line of
/root/reference/pkg/src/phraseboost/):
  * score_batch / ctc_greedy: ctypes bindings of oracle/pgpb_oracle.c, the
    C restatement of _kernels.pyx:30-72 and :75-225;
  * build_table: pure-Python trie + fail links + arc table
    (tree.py:145-214, table.py:138-187), returning the reference's arrays;
  * ctc_greedy_decode, ctc_beam, transducer_greedy, transducer_beam,
    aed_beam: restatements of decoding.py:156-587 (R6-R12 of SURVEY.md);
  * ref_kernels(): the reference's *own* Cython module compiled into
    oracle/_ref/ (oracle/build_ref.py), when present.

Pinned against golden vectors produced by the reference itself
(tests/golden/gen_golden.py); see tests/test_oracle.py.
"""

from __future__ import annotations

import ctypes
import importlib.util
import math
import subprocess
from collections import deque
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "lib" / "liboracle.so"
NEG_INF = float("-inf")


def build() -> Path:
    """Compile pgpb_oracle.c (gcc) if needed."""
    src = HERE / "pgpb_oracle.c"
    if not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-C", str(HERE), "lib/liboracle.so"], check=True, capture_output=True)
    return LIB_PATH


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(LIB_PATH))
        P = ctypes.c_void_p
        L.oracle_score_batch.argtypes = [P] * 9 + [ctypes.c_int64, P, ctypes.c_int64, P, P]
        L.oracle_score_batch.restype = ctypes.c_int
        L.oracle_ctc_greedy.argtypes = [P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_double,
                                        ctypes.c_int32] + [P] * 9 + [P] * 5
        L.oracle_ctc_greedy.restype = ctypes.c_int64
        _lib = L
    return _lib


def _p(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def _tab_arrays(t):
    c = np.ascontiguousarray
    return [c(t.arc_token, np.int32), c(t.arc_to, np.int32), c(t.arc_weight, np.float32),
            c(t.state_start, np.int32), c(t.state_end, np.int32), c(t.backoff_to, np.int32),
            c(t.backoff_weight, np.float32), c(t.root_scores, np.float32), c(t.root_next, np.int32)]


def score_batch(table, states) -> tuple[np.ndarray, np.ndarray]:
    """_kernels.pyx:30-72 on any object carrying the reference ArcTable arrays."""
    st = np.ascontiguousarray(np.asarray(states, dtype=np.int32).reshape(-1))
    V = int(table.vocab_size)
    scores = np.empty((st.shape[0], V), np.float32)
    nxt = np.empty((st.shape[0], V), np.int32)
    arrs = _tab_arrays(table)
    rc = lib().oracle_score_batch(*[_p(a) for a in arrs], V, _p(st), st.shape[0], _p(scores), _p(nxt))
    assert rc == 0
    return scores, nxt


def ctc_greedy(logprobs: np.ndarray, blank: int, lam: float, use_boost: bool, table):
    """_kernels.pyx:75-225: (tokens, am, boost, deltas, states)."""
    lp = np.ascontiguousarray(logprobs, dtype=np.float32)
    T, V = lp.shape
    if table is None:
        arrs = [np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros(0, np.float32),
                np.zeros(1, np.int32), np.zeros(1, np.int32), np.zeros(1, np.int32),
                np.zeros(1, np.float32), np.zeros(V, np.float32), np.zeros(V, np.int32)]
        use_boost = False
    else:
        arrs = _tab_arrays(table)
    tok = np.empty(max(T, 1), np.int32)
    dl = np.empty(max(T, 1), np.float64)
    stt = np.empty(max(T, 1), np.int32)
    am = ctypes.c_double()
    bo = ctypes.c_double()
    n = lib().oracle_ctc_greedy(_p(lp), T, V, int(blank), float(lam), int(bool(use_boost)),
                                *[_p(a) for a in arrs], _p(tok), _p(dl), _p(stt),
                                ctypes.byref(am), ctypes.byref(bo))
    assert n >= 0
    return tok[:n].copy(), am.value, bo.value, dl[:n].copy(), stt[:n].copy()


def ref_kernels():
    """The reference's own compiled module from oracle/_ref/, or None."""
    d = HERE / "_ref"
    cands = sorted(d.glob("_kernels*.so")) if d.exists() else []
    if not cands:
        return None
    spec = importlib.util.spec_from_file_location("_kernels", cands[0])
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


# ---------------------------------------------------------------------------
# Tree build restatement (tree.py:145-214, table.py:138-187)


@dataclass
class OracleTable:
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
    acc: np.ndarray | None = None
    root_scores: np.ndarray = field(init=False)
    root_next: np.ndarray = field(init=False)

    def __post_init__(self):  # table.py:74-81
        self.root_scores = np.full(self.vocab_size, np.float32(self.unk_score), np.float32)
        self.root_next = np.zeros(self.vocab_size, np.int32)
        lo, hi = int(self.state_start[0]), int(self.state_end[0])
        self.root_scores[self.arc_token[lo:hi]] = self.arc_weight[lo:hi]
        self.root_next[self.arc_token[lo:hi]] = self.arc_to[lo:hi]


def _arc_score(depth, c0, beta, mode):  # tree.py:53-61
    if mode == "uniform" or depth == 1:
        return c0
    return c0 * beta + math.log(depth)


def build_table(phrases, V, c0=1.0, beta=2.0, mode="depth_scaled", bonus=0.0, unk=0.0) -> OracleTable:
    """phrases: sequence of token-id tuples in ContextList order."""
    parent, depth, in_tok, final = [-1], [0], [-1], [False]
    arcs: list[dict[int, int]] = [{}]
    for ph in phrases:  # tree.py:155-172
        if not ph:
            raise ValueError("empty phrase")
        cur = 0
        for tkn in ph:
            if not 0 <= tkn < V:
                raise ValueError("token out of range")
            nxt = arcs[cur].get(tkn)
            if nxt is None:
                nxt = len(parent)
                parent.append(cur)
                depth.append(depth[cur] + 1)
                in_tok.append(tkn)
                final.append(False)
                arcs.append({})
                arcs[cur][tkn] = nxt
            cur = nxt
        final[cur] = True
    S = len(parent)
    score = [0.0] * S
    acc = [0.0] * S
    for i in range(1, S):  # tree.py:175-184
        s = _arc_score(depth[i], c0, beta, mode)
        if mode == "uniform" and final[i]:
            s += bonus
        score[i] = s
        acc[i] = acc[parent[i]] + s
    fail = [0] * S  # tree.py:196-213
    q = deque()
    for tkn in sorted(arcs[0]):
        q.append(arcs[0][tkn])
    while q:
        nid = q.popleft()
        for tkn in sorted(arcs[nid]):
            ch = arcs[nid][tkn]
            f = fail[nid]
            while f != 0 and tkn not in arcs[f]:
                f = fail[f]
            hit = arcs[f].get(tkn)
            fail[ch] = hit if hit is not None and hit != ch else 0
            q.append(ch)
    rows = sorted((p, in_tok[c], c, score[c]) for c, p in enumerate(parent) if c)
    A = len(rows)
    arc_from = np.array([r[0] for r in rows], np.int32).reshape(-1)
    arc_token = np.array([r[1] for r in rows], np.int32).reshape(-1)
    arc_to = np.array([r[2] for r in rows], np.int32).reshape(-1)
    arc_weight = np.array([r[3] for r in rows], np.float64).reshape(-1).astype(np.float32)
    ss = np.searchsorted(arc_from, np.arange(S), side="left").astype(np.int32)
    se = np.searchsorted(arc_from, np.arange(S), side="right").astype(np.int32)
    acc_a = np.array(acc, np.float64)
    bt = np.array(fail, np.int32)
    fin = np.array(final, bool)
    bw = (acc_a[bt] - acc_a).astype(np.float32)  # table.py:163-169
    bw[fin] = 0.0
    bw[0] = 0.0
    fs = np.where(fin, acc_a, 0.0).astype(np.float32)
    assert A == S - 1
    return OracleTable(S, V, arc_from, arc_token, arc_to, arc_weight, ss, se, bt, bw, fin, fs,
                       float(unk), acc=acc_a)


# ---------------------------------------------------------------------------
# Decoder restatements (decoding.py).  Results: dicts with tokens, am,
# boost, trace [(token, delta, state)].


def _logaddexp(a: float, b: float) -> float:  # decoding.py:94-100
    if a == NEG_INF:
        return b
    if b == NEG_INF:
        return a
    m = a if a > b else b
    return m + math.log1p(math.exp(-abs(a - b)))


def _rerank(row, srow, lam, exclude) -> int:  # decoding.py:129-149
    comb = row.astype(np.float64) + np.float64(lam) * srow.astype(np.float64)
    for v in exclude:
        if v >= 0:
            comb[v] = NEG_INF
    best = comb.max()
    cand = np.flatnonzero(comb == best)
    if cand.size > 1:
        raws = row[cand]
        cand = cand[raws == raws.max()]
    return int(cand[0])


def _active(table, lam, enabled=True) -> bool:  # decoding.py:103-104
    return table is not None and enabled and lam != 0.0


def ctc_greedy_decode(lp, blank, table, lam, enabled=True):
    """decoding.py:156-229 through the C restatement of the compiled kernel."""
    use = _active(table, lam, enabled)
    tok, am, bo, dl, st = ctc_greedy(lp, blank, lam, use, table if use else None)
    return {"tokens": [int(x) for x in tok], "am": am, "boost": bo,
            "trace": [(int(a), float(b), int(c)) for a, b, c in zip(tok, dl, st)]}


def ctc_greedy_numpy(lp, blank, table, lam, enabled=True):
    """decoding.py:200-229 (the reference's NumPy path), independent of the C kernel."""
    use = _active(table, lam, enabled)
    raw = np.argmax(lp, axis=1)
    toks, trace = [], []
    am = boost = 0.0
    last, state = -1, 0
    for t in range(lp.shape[0]):
        a = int(raw[t])
        if a == blank or a == last:
            am += float(lp[t, a])
            last = a
            continue
        if use:
            sc, nx = score_batch(table, [state])
            ch = _rerank(lp[t], sc[0], lam, (blank, last))
            d, ns = float(sc[0, ch]), int(nx[0, ch])
        else:
            ch, d, ns = a, 0.0, 0
        toks.append(ch)
        trace.append((ch, d, ns))
        am += float(lp[t, ch])
        boost += d
        state, last = ns, ch
    return {"tokens": toks, "am": am, "boost": boost, "trace": trace}


def ctc_beam(lp, blank, table, lam, beam, enabled=True, rollback=False):
    """Prefix beam search, decoding.py:247-343 (R8).  Returns n-best dicts.

    rollback=True is an extension with NO reference counterpart (parity
    unpinned): after the last frame every prefix gets backoff_total(state)
    added to its boost before the final ranking."""
    use = _active(table, lam, enabled)
    T, V = lp.shape
    # prefix -> [pb, pnb, state, boost, trace]
    entries = {(): [0.0, NEG_INF, 0, 0.0, ()]}
    for t in range(T):
        items = list(entries.items())
        if use:
            sc, nx = score_batch(table, [e[2] for _, e in items])
        new = {}

        def carry(prefix, e):
            ne = new.get(prefix)
            if ne is None:
                ne = [NEG_INF, NEG_INF, e[2], e[3], e[4]]
                new[prefix] = ne
            return ne

        for i, (prefix, e) in enumerate(items):
            tot = _logaddexp(e[0], e[1])
            ne = carry(prefix, e)
            ne[0] = _logaddexp(ne[0], tot + float(lp[t, blank]))
            last = prefix[-1] if prefix else -1
            for v in range(V):
                if v == blank:
                    continue
                lv = float(lp[t, v])
                if v == last:
                    ne[1] = _logaddexp(ne[1], e[1] + lv)
                    contrib = e[0] + lv
                else:
                    contrib = tot + lv
                if contrib == NEG_INF:
                    continue
                newp = prefix + (v,)
                ne2 = new.get(newp)
                if ne2 is None:
                    if use:
                        d, ns = float(sc[i, v]), int(nx[i, v])
                    else:
                        d, ns = 0.0, 0
                    ne2 = [NEG_INF, NEG_INF, ns, e[3] + d, e[4] + ((v, d, ns),)]
                    new[newp] = ne2
                ne2[1] = _logaddexp(ne2[1], contrib)
        ranked = sorted(new.items(), key=lambda kv: (-(_logaddexp(kv[1][0], kv[1][1]) + lam * kv[1][3]),
                                                     -_logaddexp(kv[1][0], kv[1][1]), kv[0]))
        entries = dict(ranked[:beam])
    if rollback and use and T > 0:
        entries = {p: [e[0], e[1], e[2], e[3] + backoff_total(table, e[2]), e[4]] for p, e in entries.items()}
    ranked = sorted(entries.items(), key=lambda kv: (-(_logaddexp(kv[1][0], kv[1][1]) + lam * kv[1][3]),
                                                     -_logaddexp(kv[1][0], kv[1][1]), kv[0]))
    return [{"tokens": list(p), "am": _logaddexp(e[0], e[1]), "boost": e[3], "trace": list(e[4])}
            for p, e in ranked[:beam]]


def transducer_greedy(step, T, blank, table, lam, max_symbols, enabled=True):
    """decoding.py:350-393 (R7).  step(last_token_or_None, t) -> f32 row."""
    use = _active(table, lam, enabled)
    toks, trace = [], []
    am = boost = 0.0
    state, last = 0, None
    for t in range(T):
        for _ in range(max_symbols):
            row = step(last, t)
            a = int(np.argmax(row))
            if a == blank:
                am += float(row[blank])
                break
            if use:
                sc, nx = score_batch(table, [state])
                ch = _rerank(row, sc[0], lam, (blank,))
                d, ns = float(sc[0, ch]), int(nx[0, ch])
            else:
                ch, d, ns = a, 0.0, 0
            toks.append(ch)
            trace.append((ch, d, ns))
            am += float(row[ch])
            boost += d
            state, last = ns, ch
    return {"tokens": toks, "am": am, "boost": boost, "trace": trace}


def transducer_greedy_tdt(step, T, blank, table, lam, max_symbols, enabled=True):
    """TDT greedy (no reference counterpart; the label-looping kernel's rules):
    step(last_token_or_None, t) -> (f32 row, duration).  Token decisions are
    R7's (argmax, blank test, boosted rerank excluding blank); a blank adds its
    log-prob and advances max(d, 1) frames; an emission advances d frames
    (d > 0) or stays (d == 0) until max_symbols emissions, then advances 1.
    With d = 1 on blanks and d = 0 on emissions this is transducer_greedy."""
    use = _active(table, lam, enabled)
    toks, trace = [], []
    am = boost = 0.0
    state, last = 0, None
    t, k = 0, 0
    while t < T:
        row, dur = step(last, t)
        a = int(np.argmax(row))
        if a == blank:
            am += float(row[blank])
            t += max(int(dur), 1)
            k = 0
            continue
        if use:
            sc, nx = score_batch(table, [state])
            ch = _rerank(row, sc[0], lam, (blank,))
            d, ns = float(sc[0, ch]), int(nx[0, ch])
        else:
            ch, d, ns = a, 0.0, 0
        toks.append(ch)
        trace.append((ch, d, ns))
        am += float(row[ch])
        boost += d
        state, last = ns, ch
        k += 1
        if dur > 0:
            t += int(dur)
            k = 0
        elif k >= max_symbols:
            t += 1
            k = 0
    return {"tokens": toks, "am": am, "boost": boost, "trace": trace}


@dataclass
class _Hyp:
    tokens: tuple
    am: float
    boost: float
    state: int
    last: int | None = None
    ended: bool = False
    trace: tuple = ()


def _keep_better(pool, key, cand, lam):  # decoding.py:396-404
    old = pool.get(key)
    if old is None or (cand.am + lam * cand.boost, cand.am) > (old.am + lam * old.boost, old.am):
        pool[key] = cand


def _rank(lam):  # decoding.py:407-411
    return lambda h: (-(h.am + lam * h.boost), -h.am, h.tokens)


def _out(beam, lam, k):
    return [{"tokens": list(h.tokens), "am": h.am, "boost": h.boost, "trace": list(h.trace)}
            for h in sorted(beam, key=_rank(lam))[:k]]


def backoff_total(table, s: int) -> float:
    """fp32 sum of backoff weights along s's chain, in chain order (_kernels.pyx:59-66)."""
    acc = np.float32(0.0)
    while s != 0:
        acc = np.float32(acc + np.float32(table.backoff_weight[s]))
        s = int(table.backoff_to[s])
    return float(acc)


def transducer_beam(step, T, blank, table, lam, beam_size, max_symbols, V, enabled=True, rollback=False):
    """decoding.py:428-495 (R9).

    rollback=True is an extension with NO reference counterpart (parity
    unpinned): at the last frame every finished hypothesis gets
    backoff_total(state) added to its boost before the final pruning.
    """
    use = _active(table, lam, enabled)
    rank = _rank(lam)
    beam = [_Hyp((), 0.0, 0.0, 0)]
    for t in range(T):
        active = {}
        for h in beam:
            _keep_better(active, (h.tokens, 0), h, lam)
        finished = {}
        while active:
            waves = sorted(active.items(), key=lambda kv: rank(kv[1]))
            if use:
                sc, nx = score_batch(table, [h.state for _, h in waves])
            nxt = {}
            for i, ((toks, k), h) in enumerate(waves):
                row = step(h.last, t)
                bh = _Hyp(h.tokens, h.am + float(row[blank]), h.boost, h.state, h.last, h.ended, h.trace)
                _keep_better(finished, bh.tokens, bh, lam)
                if k >= max_symbols:
                    continue
                for v in range(V):
                    if v == blank:
                        continue
                    d, ns = (float(sc[i, v]), int(nx[i, v])) if use else (0.0, 0)
                    c = _Hyp(toks + (v,), h.am + float(row[v]), h.boost + d, ns, v,
                             trace=h.trace + ((v, d, ns),))
                    _keep_better(nxt, (c.tokens, k + 1), c, lam)
            active = dict(sorted(nxt.items(), key=lambda kv: rank(kv[1]))[:beam_size])
        if rollback and use and t == T - 1:
            finished = {k: _Hyp(h.tokens, h.am, h.boost + backoff_total(table, h.state), h.state, h.last, h.ended,
                                h.trace) for k, h in finished.items()}
        beam = sorted(finished.values(), key=rank)[:beam_size]
    return _out(beam, lam, beam_size)


def aed_beam(step, table, lam, beam_size, max_len, eos, V, eos_bump=True, enabled=True, rollback=False):
    """decoding.py:502-587 (R10).  step(prefix_tuple, len) -> f32 row.

    rollback=True is an extension with NO reference counterpart (parity
    unpinned): the eos step's boost also carries backoff_total(state) (the
    unfinished phrase's credit taken back when the hypothesis ends)."""
    use = _active(table, lam, enabled)
    rank = _rank(lam)
    beam = [_Hyp((), 0.0, 0.0, 0)]
    while True:
        active = [h for h in beam if not h.ended and len(h.tokens) < max_len]
        if not active:
            break
        cands = [h for h in beam if h.ended or len(h.tokens) >= max_len]
        if use:
            sc, nx = score_batch(table, [h.state for h in active])
        for i, h in enumerate(active):
            row = step(h.tokens, len(h.tokens))
            for v in range(V):
                lv = float(row[v])
                if v == eos:
                    bump = 0.0
                    if use and eos_bump:
                        best = float(sc[i].max())
                        bump = best if best > 0.0 else 0.0
                        if bool(table.is_final[h.state]):
                            bump += float(table.final_score[h.state])
                    if use and rollback:
                        bump += backoff_total(table, h.state)
                    cands.append(_Hyp(h.tokens, h.am + lv, h.boost + bump, h.state, h.last, True,
                                      h.trace + ((eos, bump, h.state),)))
                else:
                    d, ns = (float(sc[i, v]), int(nx[i, v])) if use else (0.0, 0)
                    cands.append(_Hyp(h.tokens + (v,), h.am + lv, h.boost + d, ns, v, False,
                                      h.trace + ((v, d, ns),)))
        beam = sorted(cands, key=rank)[:beam_size]
    return _out(beam, lam, beam_size)
