"""Batched RNN-T greedy decoding with GPU-PB boosting, label-looping form.

Output-equivalent, per utterance, to the reference's frame-synchronous
greedy transducer decoder (decoding.py:350-393, R7): at frame t the
decoder keeps emitting (up to `max_symbols_per_frame`) until the stage-1
argmax is blank; a blank adds its log-prob and advances the frame; hitting
the cap advances the frame without a blank score.  Non-blank symbols are
chosen by the boosted rerank (excluding blank only) and move the tree state.

Label looping (NeMo's formulation) runs all B utterances in lock-step
"label iterations": every iteration evaluates the joint for each active
utterance at its own current frame and its own prediction-network state,
then one fused kernel (pgpb_label_loop_step: argmax, blank test, boosted
rerank, next tree state, and the whole R7 bookkeeping — scores, outputs,
frame pointers, symbol counters) decides and advances every row.  One
iteration is a fixed sequence of kernels (joint GEMMs, log-softmax, the
fused step, the LSTM cell), captured once as a CUDA graph and replayed; the
host only polls an "all done" flag every `poll` iterations.

TDT (token-and-duration transducer, NeMo's label-looping greedy): a model
built with a duration set adds a duration head; each iteration also passes
every row's duration argmax to the fused step, which advances blanks by
max(d, 1) frames and emissions by d frames (d == 0: stay, cap applies).  The
reference has no TDT, so this is a parity-unpinned extension,
checked against its own restatement (oracle.transducer_greedy_tdt), which
reduces to R7 when every emission has d = 0 and every blank d = 1.

The networks are random-init stand-ins of the paper's shapes (1-layer
LSTM-640 prediction net + joint) — library GEMMs, outside
the GPU-PB path.  Parity with the reference decoder is established by
replaying the exact log-prob rows each utterance consumed
(`record=True`) into the oracle's transducer_greedy (tests/test_rnnt_gpu.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .decoding import DecodeConfig, DecodeResult, TraceStep, _boost_active, _text
from .table import ArcTable


def _torch():
    import torch

    _lib.require_cuda()
    return torch



def _check_lengths(ln, B: int, T: int) -> None:
    """Frame counts must lie in [0, T] (the kernels index frames by them)."""
    if tuple(ln.shape) != (B,):
        raise ValueError(f"lengths must have shape ({B},), got {tuple(ln.shape)}")
    if B:
        lo, hi = (int(x) for x in ln.long().aminmax())
        if lo < 0 or hi > T:
            raise ValueError(f"lengths must lie in [0, {T}], got [{lo}, {hi}]")

class RNNTModel:
    """Random-init prediction network (Embedding + 1-layer LSTM) and joint.

    joint(enc, pred) = out(relu(enc_proj(enc) + pred_proj(pred))), then a
    float32 log-softmax over V tokens (blank included).  `blank_id` also
    serves as the start-of-sequence token of the prediction network.
    """

    def __init__(self, vocab_size: int, enc_dim: int = 512, pred_dim: int = 640, joint_dim: int = 640,
                 blank_id: int = 0, seed: int = 0, device="cuda", dtype=None, blank_bias: float = 3.0,
                 durations: tuple[int, ...] | None = None):
        """dtype defaults to bfloat16 (tensor-core GEMMs); log-probs are float32.

        durations: TDT duration set (e.g. (0, 1, 2, 3, 4)); adds a duration
        head to the joint (NeMo's token-and-duration transducer)."""
        torch = _torch()
        g = torch.Generator(device="cpu")
        g.manual_seed(seed)
        dt = dtype or torch.bfloat16
        V, D, H, J = vocab_size, enc_dim, pred_dim, joint_dim

        def w(*shape, fan_in):
            return (torch.randn(*shape, generator=g) / np.sqrt(fan_in)).to(device=device, dtype=dt)

        self.V, self.D, self.H, self.J, self.blank_id = V, D, H, J, blank_id
        self.dtype = dt
        self.emb = w(V, H, fan_in=1.0) * 0.5
        self.w_ih = w(4 * H, H, fan_in=H)
        self.w_hh = w(4 * H, H, fan_in=H)
        self.b_lstm = torch.zeros(4 * H, device=device, dtype=dt)
        self.b_hh = torch.zeros(4 * H, device=device, dtype=dt)
        self.w_enc = w(J, D, fan_in=D)
        self.w_pred = w(J, H, fan_in=H)
        self.b_joint = torch.zeros(J, device=device, dtype=dt)
        self.w_out = w(V, J, fan_in=J) * 3.0  # peaky enough for confident argmaxes
        self.b_out = torch.zeros(V, device=device, dtype=dt)
        self.b_out[blank_id] = blank_bias  # blank-dominated frames, as trained transducers are
        self.durations = tuple(int(d) for d in durations) if durations else None
        if self.durations:
            if min(self.durations) < 0:
                raise ValueError("durations must be >= 0")
            self.w_dur = w(len(self.durations), J, fan_in=J) * 3.0
            self.dur_values = torch.tensor(self.durations, device=device, dtype=torch.int32)
        # input gates of every token, emb @ W_ih^T + b_ih (one GEMM per model):
        # a prediction step then gathers its row instead of embedding + GEMM
        self.E = torch.addmm(self.b_lstm, self.emb, self.w_ih.T) if dt == torch.bfloat16 else None
        # both GEMMs that read the prediction state h, stacked: one GEMM per
        # label iteration gives [pred_proj | hidden gates]
        self.w_cat = torch.cat([self.w_pred, self.w_hh], 0)
        self.b_cat = torch.cat([self.b_joint, self.b_hh], 0)

    def project_encoder(self, enc):
        """enc [B,T,D] -> [B,T,J] (computed once per batch)."""
        return enc.to(self.dtype) @ self.w_enc.T

    def lstm_step(self, tokens, h, c):
        """One prediction-network step for tokens [B] (int64)."""
        torch = _torch()
        x = self.emb.index_select(0, tokens)
        return torch.lstm_cell(x, (h, c), self.w_ih, self.w_hh, self.b_lstm, self.b_hh)

    def joint_logprobs(self, enc_proj_t, pred_h):
        """[B,J] encoder projection at each row's frame + [B,H] -> [B,V] float32 log-probs."""
        return self.joint(enc_proj_t, pred_h)[0]

    def joint(self, enc_proj_t, pred_h):
        """Token log-probs [B,V] f32 and, for TDT, each row's duration (argmax of
        the duration head, first max) as int32 frames; None for RNN-T."""
        torch = _torch()
        z = torch.relu(enc_proj_t + torch.addmm(self.b_joint, pred_h, self.w_pred.T))
        logits = torch.addmm(self.b_out, z, self.w_out.T)
        lp = torch.log_softmax(logits.float(), dim=-1)
        if not self.durations:
            return lp, None
        dl = (z @ self.w_dur.T).float()
        return lp, self.dur_values[torch.argmax(dl, dim=-1)]


@dataclass
class LabelLoopOutput:
    tokens: object      # int32 [B, Lmax]
    deltas: object      # float64 [B, Lmax]
    states: object      # int32 [B, Lmax]
    num_out: object     # int32 [B]
    am: object          # float64 [B]
    boost: object       # float64 [B]
    iterations: int
    records: list | None = None  # per iteration (lp[B,V], active[B], t[B], last[B]) when record=True


class LabelLoopingDecoder:
    """Batched boosted greedy RNN-T decoder over a fixed batch geometry.

    Build once per (model, table, cfg, B, T); `decode(enc_proj, lengths)`
    resets the state tensors in place and replays the captured iteration
    graph until every utterance has consumed its frames.
    """

    def __init__(self, model: RNNTModel, table: ArcTable | None, cfg: DecodeConfig, batch: int, max_frames: int,
                 *, use_graph: bool = True, poll: int = 16, device=None, fused: bool = True):
        torch = _torch()
        self.torch = torch
        self.model, self.table, self.cfg = model, table, cfg
        self.B, self.T, self.V = batch, max_frames, model.V
        if table is not None and table.vocab_size != model.V:
            raise ValueError(f"step model vocab size {model.V} != table vocab size {table.vocab_size}")
        self.use = _boost_active(table, cfg)
        self.dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.handle = table.device_table(self.dev.index).handle if self.use else None
        self.cap = cfg.max_symbols_per_frame
        self.Lmax = max_frames * self.cap
        self.poll = poll
        self.use_graph = use_graph
        B, d = batch, self.dev
        i32, i64, f32, f64 = torch.int32, torch.int64, torch.float32, torch.float64
        # persistent state (addresses fixed for the graph)
        self.enc_proj = torch.zeros((B, max_frames, model.J), device=d, dtype=model.dtype)
        self.lengths = torch.zeros(B, device=d, dtype=i64)
        self.t = torch.zeros(B, device=d, dtype=i64)
        self.k = torch.zeros(B, device=d, dtype=i64)
        self.last = torch.full((B,), model.blank_id, device=d, dtype=i64)
        self.h = torch.zeros((B, model.H), device=d, dtype=model.dtype)
        self.c = torch.zeros((B, model.H), device=d, dtype=model.dtype)
        self.tree = torch.zeros(B, device=d, dtype=i32)
        self.tree_off = torch.full((B,), -1, device=d, dtype=i32)  # blob offset of tree (-1: look up)
        self.am = torch.zeros(B, device=d, dtype=f64)
        self.boost = torch.zeros(B, device=d, dtype=f64)
        self.n = torch.zeros(B, device=d, dtype=i64)
        self.tokens = torch.zeros((B, self.Lmax), device=d, dtype=i32)
        self.deltas = torch.zeros((B, self.Lmax), device=d, dtype=f64)
        self.states = torch.zeros((B, self.Lmax), device=d, dtype=i32)
        self.emit = torch.zeros(B, device=d, dtype=torch.uint8)
        self.feed = torch.zeros(B, device=d, dtype=i64)
        self.lp = torch.zeros((B, model.V), device=d, dtype=f32)
        self.dur = torch.zeros(B, device=d, dtype=i32) if model.durations else None
        self.any_active = torch.zeros(1, device=d, dtype=i32)
        self.flag_host = torch.zeros(1, dtype=i32, pin_memory=True)
        self.rows = torch.arange(B, device=d)
        # fused kernels for RNN-T (bf16 networks); TDT keeps the framework path
        self.fused = fused and model.durations is None and model.E is not None
        self.z = torch.zeros((B, model.J), device=d, dtype=model.dtype)
        self.graph = None
        p = lambda x: x.data_ptr()  # noqa: E731
        self.state = _lib.LabelLoopState(p(self.t), p(self.k), p(self.lengths), p(self.n), p(self.last), p(self.tree),
                                         p(self.am), p(self.boost), p(self.tokens), p(self.deltas), p(self.states),
                                         self.Lmax, self.cap, p(self.dur) if self.dur is not None else None,
                                         p(self.tree_off))

    # -- one label iteration (fixed kernel sequence) ------------------------
    def _iteration(self):
        if self.fused:
            return self._iteration_fused()
        torch, m = self.torch, self.model
        self.any_active.zero_()
        tf = torch.minimum(self.t, (self.lengths - 1).clamp(min=0))
        lp, dur = m.joint(self.enc_proj[self.rows, tf], self.h)
        self.lp.copy_(lp)
        if dur is not None:
            self.dur.copy_(dur)
        _lib.check(_lib.LIB.pgpb_label_loop_step(
            self.handle, self.lp.data_ptr(), self.V, self.B, self.V, int(m.blank_id), float(self.cfg.lam),
            int(self.use), _lib.ctypes.byref(self.state), self.emit.data_ptr(), self.feed.data_ptr(),
            self.any_active.data_ptr(), _lib.stream_ptr(),
        ), "pgpb_label_loop_step")
        # the prediction network advances on emitted tokens only
        h2, c2 = m.lstm_step(self.feed, self.h, self.c)
        e2 = self.emit.bool().unsqueeze(1)
        self.h.copy_(torch.where(e2, h2, self.h))
        self.c.copy_(torch.where(e2, c2, self.c))

    def _iteration_fused(self):
        """The same iteration as 2 bf16 GEMMs + 3 kernels: one GEMM of h against
        the stacked [W_pred; W_hh], joint hidden (frame gather + add + ReLU),
        the output GEMM, log-softmax fused into the boosted step
        (pgpb_label_loop_step_logits, which writes self.lp), and the LSTM cell
        on the precomputed input gates, updating h, c of emitting rows."""
        torch, m = self.torch, self.model
        self.any_active.zero_()
        ph = torch.addmm(m.b_cat, self.h, m.w_cat.T)  # [B, J + 4H]: pred projection | hidden gates
        ld = m.J + 4 * m.H
        _lib.check(_lib.LIB.pgpb_rnnt_joint_hidden(
            self.enc_proj.data_ptr(), self.T * m.J, m.J, self.t.data_ptr(), self.lengths.data_ptr(), ph.data_ptr(),
            ld, self.z.data_ptr(), self.B, _lib.stream_ptr()), "pgpb_rnnt_joint_hidden")
        logits = torch.addmm(m.b_out, self.z, m.w_out.T)
        _lib.check(_lib.LIB.pgpb_label_loop_step_logits(
            self.handle, logits.data_ptr(), self.V, self.lp.data_ptr(), self.B, self.V, int(m.blank_id),
            float(self.cfg.lam), int(self.use), _lib.ctypes.byref(self.state), self.emit.data_ptr(),
            self.feed.data_ptr(), self.any_active.data_ptr(), _lib.stream_ptr(),
        ), "pgpb_label_loop_step_logits")
        _lib.check(_lib.LIB.pgpb_rnnt_lstm_update(
            m.E.data_ptr(), self.feed.data_ptr(), ph.data_ptr() + 2 * m.J, ld, self.emit.data_ptr(),
            self.h.data_ptr(), self.c.data_ptr(), self.B, m.H, _lib.stream_ptr()), "pgpb_rnnt_lstm_update")

    def _reset(self, enc_proj, lengths):
        torch = self.torch
        B, T = enc_proj.shape[0], enc_proj.shape[1]
        if B != self.B or T > self.T:
            raise ValueError("batch geometry differs from the decoder's")
        self.enc_proj[:, :T].copy_(enc_proj)
        ln = torch.as_tensor(lengths, device=self.dev).long() if lengths is not None else torch.full(
            (B,), T, device=self.dev, dtype=torch.int64)
        _check_lengths(ln, B, T)
        self.lengths.copy_(ln)
        for x in (self.t, self.k, self.n, self.am, self.boost, self.tree, self.h, self.c):
            x.zero_()
        self.last.fill_(self.model.blank_id)
        self.tree_off.fill_(-1)
        # initial prediction state: one step on the start symbol (blank)
        if self.fused:
            m = self.model
            hg = torch.addmm(m.b_hh, self.h, m.w_hh.T)
            _lib.check(_lib.LIB.pgpb_rnnt_lstm_update(
                m.E.data_ptr(), self.last.data_ptr(), hg.data_ptr(), 4 * m.H, None, self.h.data_ptr(),
                self.c.data_ptr(), self.B, m.H, _lib.stream_ptr()), "pgpb_rnnt_lstm_update")
            return
        h2, c2 = self.model.lstm_step(self.last, self.h, self.c)
        self.h.copy_(h2)
        self.c.copy_(c2)

    def _capture(self):
        torch = self.torch
        s = torch.cuda.Stream(self.dev)
        s.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(s):  # warm-up allocations outside the capture
            self._iteration()
        torch.cuda.current_stream(self.dev).wait_stream(s)
        # one poll interval of iterations per graph: one launch per host check
        # (iterations past the end are no-ops on finished rows)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(self.poll):
                self._iteration()
        self.graph = g

    def decode(self, enc_proj, lengths=None, *, record: bool = False, max_iters: int | None = None) -> LabelLoopOutput:
        torch = self.torch
        if self.use_graph and self.graph is None and not record:
            self._reset(enc_proj, lengths)
            self._capture()
        self._reset(enc_proj, lengths)
        limit = max_iters or (self.T * (self.cap + 1) + 1)
        records = [] if record else None
        it = 0
        while it < limit:
            steps = min(self.poll, limit - it)
            graphed = self.graph is not None and not record and steps == self.poll
            if graphed:
                self.graph.replay()  # self.poll iterations
            for _ in range(0 if graphed else steps):
                if record:
                    t0, last0 = self.t.clone(), self.last.clone()
                    active = (t0 < self.lengths).cpu().numpy()
                    self._iteration()
                    rec = (self.lp.cpu().numpy().copy(), active, t0.cpu().numpy(), last0.cpu().numpy())
                    if self.dur is not None:
                        rec = rec + (self.dur.cpu().numpy().copy(),)
                    records.append(rec)
                else:
                    self._iteration()
            it += steps
            self.flag_host.copy_(self.any_active, non_blocking=True)
            torch.cuda.current_stream(self.dev).synchronize()
            if int(self.flag_host[0]) == 0:
                break
        return LabelLoopOutput(self.tokens, self.deltas, self.states, self.n.int(), self.am, self.boost, it, records)


def transducer_greedy_label_looping(model: RNNTModel, enc, lengths=None, table: ArcTable | None = None,
                                    cfg: DecodeConfig | None = None, *, vocab=None, want_trace: bool = False,
                                    use_graph: bool = True) -> list[DecodeResult]:
    """Batched boosted greedy RNN-T over enc [B,T,D]; per-utterance DecodeResults."""
    cfg = cfg or DecodeConfig()
    B, T = enc.shape[0], enc.shape[1]
    dec = LabelLoopingDecoder(model, table, cfg, B, T, use_graph=use_graph)
    o = dec.decode(model.project_encoder(enc), lengths)
    n = o.num_out.cpu().numpy()
    tok, dl, st = o.tokens.cpu().numpy(), o.deltas.cpu().numpy(), o.states.cpu().numpy()
    am, bo = o.am.cpu().numpy(), o.boost.cpu().numpy()
    out = []
    for b in range(B):
        k = int(n[b])
        tokens = [int(x) for x in tok[b, :k]]
        trace = [TraceStep(int(x), float(y), int(z)) for x, y, z in zip(tok[b, :k], dl[b, :k], st[b, :k])] \
            if want_trace else None
        out.append(DecodeResult(tokens, _text(tokens, vocab), float(am[b]), float(bo[b]), trace))
    return out
