"""Batched device-resident beam search with GPU-PB boosting.

The reference's beam decoders (decoding.py:428-495 transducer, R9;
decoding.py:502-587 AED, R10) keep hypotheses in Python dicts and loop over
the vocabulary per hypothesis, one utterance at a time.  Here a whole batch
of utterances decodes in lock-step on the GPU and the hypothesis bookkeeping
— per-hypothesis tree states, boost accumulation, merges by token sequence
(_keep_better), pruning to the beam, the AED eos bump and the opt-in
end-of-utterance rollback of unfinished phrases — runs inside the fused
expansion + top-k kernels (pgpb_tbeam_wave / pgpb_aed_step, csrc/pgpb_dbeam.cu).
The host only launches a fixed kernel sequence per frame (transducer: one
CUDA graph per frame) or per label step (AED).

Token sequences live in an append-only device trie of trace nodes
(pgpb_beam_trace); results are read back once at the end.

The networks are random-init stand-ins of the paper's shapes (outside the
GPU-PB path, library GEMMs): a stateless (last-token) transducer prediction
network + joint — the context the reference StepModel contract defines for
transducers (acoustic.py:206-208) — and a 4-layer transformer decoder
(d=256, FF 1024) with KV caches reordered by the kernel's parent slots.
Parity with the reference decoders is checked by replaying the exact rows the
GPU consumed into the oracle (tests/test_dbeam_gpu.py).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .decoding import DecodeConfig, DecodeResult, TraceStep, _boost_active, _text
from .rnnt import _check_lengths
from .table import ArcTable

VALID, ENDED = 1, 2


def _torch():
    import torch

    _lib.require_cuda()
    return torch


class _Hyps:
    """pgpb_beam_hyps buffers, [B, K] each."""

    def __init__(self, torch, B, K, dev):
        i32, f64 = torch.int32, torch.float64
        self.am = torch.zeros((B, K), dtype=f64, device=dev)
        self.boost = torch.zeros((B, K), dtype=f64, device=dev)
        self.tree = torch.zeros((B, K), dtype=i32, device=dev)
        self.last = torch.zeros((B, K), dtype=i32, device=dev)
        self.node = torch.zeros((B, K), dtype=i32, device=dev)
        self.len = torch.zeros((B, K), dtype=i32, device=dev)
        self.hash = torch.zeros((B, K), dtype=torch.int64, device=dev)  # uint64 bits
        self.flags = torch.zeros((B, K), dtype=torch.uint8, device=dev)
        self.parent = torch.zeros((B, K), dtype=i32, device=dev)

    def reset(self):
        for x in (self.am, self.boost, self.tree, self.len, self.hash, self.flags):
            x.zero_()
        self.last.fill_(-1)
        self.node.fill_(-1)
        self.flags[:, 0] = VALID  # the empty hypothesis
        self.parent.copy_(self.parent.new_tensor(range(self.parent.shape[1])).expand_as(self.parent))

    def struct(self) -> _lib.BeamHyps:
        return _lib.BeamHyps(*(x.data_ptr() for x in (self.am, self.boost, self.tree, self.last, self.node, self.len,
                                                        self.hash, self.flags, self.parent)))

    def host(self) -> dict:
        return {k: getattr(self, k).cpu().numpy() for k in ("am", "boost", "tree", "last", "node", "len", "flags")}


class _Trace:
    """pgpb_beam_trace buffers."""

    def __init__(self, torch, B, nmax, dev):
        i32 = torch.int32
        self.nmax = nmax
        self.parent = torch.zeros((B, nmax), dtype=i32, device=dev)
        self.token = torch.zeros((B, nmax), dtype=i32, device=dev)
        self.state = torch.zeros((B, nmax), dtype=i32, device=dev)
        self.delta = torch.zeros((B, nmax), dtype=torch.float64, device=dev)
        self.count = torch.zeros(B, dtype=i32, device=dev)
        self.overflow = torch.zeros(1, dtype=i32, device=dev)

    def reset(self):
        self.count.zero_()
        self.overflow.zero_()

    def struct(self) -> _lib.BeamTrace:
        return _lib.BeamTrace(self.parent.data_ptr(), self.token.data_ptr(), self.state.data_ptr(),
                              self.delta.data_ptr(), self.count.data_ptr(), self.overflow.data_ptr(), self.nmax)

    def host(self) -> dict:
        if int(self.overflow.item()):
            raise RuntimeError("beam trace arena overflow (increase nmax)")
        n = int(self.count.max().item()) if self.count.numel() else 0
        return {k: getattr(self, k)[:, :max(n, 1)].cpu().numpy() for k in ("parent", "token", "state", "delta")}


def _walk(tr: dict, b: int, node: int):
    steps = []
    while node >= 0:
        steps.append((int(tr["token"][b, node]), float(tr["delta"][b, node]), int(tr["state"][b, node])))
        node = int(tr["parent"][b, node])
    steps.reverse()
    return steps


def _collect(hy: dict, tr: dict, b: int, lam: float, vocab, want_trace: bool, eos: int | None = None):
    """n-best DecodeResults of utterance b, ranked by R11 (decoding.py:407-425)."""
    out = []
    for r in range(hy["flags"].shape[1]):
        f = int(hy["flags"][b, r])
        if not f & VALID:
            continue
        steps = _walk(tr, b, int(hy["node"][b, r]))
        toks = [s[0] for s in steps]
        if f & ENDED and eos is not None:
            toks = toks[:-1]  # the eos step is in the trace, not in the tokens
        out.append((toks, float(hy["am"][b, r]), float(hy["boost"][b, r]), steps))
    out.sort(key=lambda x: (-(x[1] + lam * x[2]), -x[1], tuple(x[0])))
    return [DecodeResult(list(t), _text(t, vocab), a, bo, [TraceStep(*s) for s in st] if want_trace else None)
            for t, a, bo, st in out]


# ---------------------------------------------------------------------------
# Transducer (config 3)


class StatelessTransducerModel:
    """Random-init stateless prediction network + joint (V outputs, blank included).

    The prediction network sees only the last emitted token (context 1, as
    NeMo's stateless decoder and the reference StepModel contract), so
    pred(last) is a [V, J] table computed once:
        row(last, t) = log_softmax(out(relu(enc_proj[t] + predJ[last])))
    `blank_id` doubles as the start symbol.
    """

    def __init__(self, vocab_size: int, enc_dim: int = 512, pred_dim: int = 640, joint_dim: int = 640,
                 blank_id: int = 0, seed: int = 0, device="cuda", dtype=None, blank_bias: float = 3.0):
        torch = _torch()
        g = torch.Generator(device="cpu")
        g.manual_seed(seed)
        dt = dtype or torch.bfloat16
        V, D, H, J = vocab_size, enc_dim, pred_dim, joint_dim

        def w(*shape, fan_in):
            return (torch.randn(*shape, generator=g) / np.sqrt(fan_in)).to(device=device, dtype=dt)

        self.V, self.D, self.H, self.J, self.blank_id, self.dtype = V, D, H, J, blank_id, dt
        self.emb = w(V, H, fan_in=1.0) * 0.5
        self.w_enc = w(J, D, fan_in=D)
        self.w_pred = w(J, H, fan_in=H)
        self.w_out = w(V, J, fan_in=J) * 3.0
        self.b_out = torch.zeros(V, device=device, dtype=dt)
        self.b_out[blank_id] = blank_bias
        self.pred_j = self.emb @ self.w_pred.T  # [V, J]

    def project_encoder(self, enc):
        return enc.to(self.dtype) @ self.w_enc.T

    def align(self, beta: float = 3.0, gamma: float = 1.0):
        """Structured init of the prediction table for a transducer-like
        alignment behaviour (benchmarks): every context adds beta * relu(w_out
        [blank]) to the joint hidden (blank likely once the frame's token has
        been emitted) and a token context subtracts gamma * w_out[token]
        (repeating it is unlikely), so a frame that favours token y emits y
        once and then blanks, as a trained transducer does.  The random part
        of the table is kept."""
        torch = _torch()
        W = self.w_out.float()
        off = beta * torch.relu(W[self.blank_id]).unsqueeze(0) - gamma * W
        off[self.blank_id] = beta * torch.relu(W[self.blank_id])
        self.pred_j = (self.pred_j.float() + off).to(self.dtype)
        return self

    def aligned_frames(self, tokens_per_frame, alpha: float = 4.0, alpha_blank: float = 2.5, noise: float = 0.1,
                       generator=None):
        """Synthetic projected encoder frames [B, T, J]: a frame with target
        token y (>= 0) is alpha * relu(w_out[y]), a blank frame (-1)
        alpha_blank * relu(w_out[blank]), plus N(0, noise)."""
        torch = _torch()
        tpf = torch.as_tensor(tokens_per_frame, device=self.w_out.device).long()
        W = torch.relu(self.w_out.float())
        idx = torch.where(tpf < 0, torch.full_like(tpf, self.blank_id), tpf)
        scale = torch.where(tpf < 0, torch.full(tpf.shape, alpha_blank, device=tpf.device),
                            torch.full(tpf.shape, alpha, device=tpf.device))
        e = W[idx] * scale.unsqueeze(-1)
        e = e + noise * torch.randn(e.shape, device=e.device, generator=generator)
        return e.to(self.dtype)

    def joint_logprobs(self, enc_t, last):
        """enc_t [B, J] (each utterance's frame), last [B, K] int (-1 = start) -> [B*K, V] f32."""
        torch = _torch()
        ctx = torch.where(last < 0, torch.full_like(last, self.blank_id), last).long()
        z = torch.relu(enc_t.unsqueeze(1) + self.pred_j[ctx])  # [B, K, J]
        logits = torch.addmm(self.b_out, z.reshape(-1, self.J), self.w_out.T)
        return torch.log_softmax(logits.float(), dim=-1)


@dataclass
class BeamOutput:
    nbest: list            # per utterance: list[DecodeResult] (best first)
    records: list | None = None


class TransducerBeamDecoder:
    """Batched boosted transducer beam search (R9) over a fixed batch geometry.

    Every frame is exactly cap + 1 waves (decoding.py:461-492: the wave loop
    ends when the per-frame symbol cap empties `active`); a wave is the joint
    for all B*beam slots followed by one pgpb_tbeam_wave launch.  One frame is
    captured as a CUDA graph and replayed max(lengths) times.
    """

    def __init__(self, model: StatelessTransducerModel, table: ArcTable | None, cfg: DecodeConfig, batch: int,
                 max_frames: int, *, use_graph: bool = True, rollback: bool | None = None, device=None,
                 fused: bool = True):
        torch = _torch()
        self.torch, self.model, self.table, self.cfg = torch, model, table, cfg
        if table is not None and table.vocab_size != model.V:
            raise ValueError(f"step model vocab size {model.V} != table vocab size {table.vocab_size}")
        if cfg.beam_size > 32:
            raise ValueError("device beam search supports beam_size <= 32")
        self.B, self.T, self.V, self.K = batch, max_frames, model.V, cfg.beam_size
        self.cap = cfg.max_symbols_per_frame
        self.use = _boost_active(table, cfg)
        self.dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.handle = table.device_table(self.dev.index).handle if self.use else None
        B, K, d = batch, self.K, self.dev
        self.pool_cap = K * (self.cap + 1)
        self.hyps = _Hyps(torch, B, K, d)
        self.pool = _Hyps(torch, B, self.pool_cap, d)
        self.pool_count = torch.zeros(B, dtype=torch.int32, device=d)
        self.trace = _Trace(torch, B, max_frames * self.cap * K + 1, d)
        self.t = torch.zeros(B, dtype=torch.int32, device=d)
        self.lengths = torch.zeros(B, dtype=torch.int32, device=d)
        self.enc_proj = torch.zeros((B, max_frames, model.J), dtype=model.dtype, device=d)
        self.lp = torch.zeros((B * K, self.V), dtype=torch.float32, device=d)
        self.rows = torch.arange(B, device=d)
        self.state = _lib.TBeamState(self.hyps.struct(), self.pool.struct(), self.pool_count.data_ptr(),
                                     self.trace.struct(), self.t.data_ptr(), self.lengths.data_ptr(), K, self.cap,
                                     self.pool_cap, int(bool(cfg.rollback if rollback is None else rollback)))
        self.use_graph = use_graph
        self.fused = fused and model.dtype == torch.bfloat16
        self.z = torch.zeros((B * K, model.J), dtype=model.dtype, device=d)
        self.graph = None
        self.launches = 0

    def _hidden(self):
        """Joint hidden rows of the current beam (frame gather + context
        gather + add + ReLU); later waves get them from the fused wave."""
        m = self.model
        _lib.check(_lib.LIB.pgpb_rnnt_beam_hidden(
            self.enc_proj.data_ptr(), self.T * m.J, m.J, self.t.data_ptr(), self.lengths.data_ptr(),
            m.pred_j.data_ptr(), self.hyps.last.data_ptr(), self.B, self.K, m.blank_id, self.z.data_ptr(),
            _lib.stream_ptr()), "pgpb_rnnt_beam_hidden")

    def _wave(self, k: int):
        torch, m = self.torch, self.model
        if self.fused:
            # a wave = the output GEMM + one kernel: log-softmax of the slots'
            # logits, the wave itself and the next wave's joint hidden rows
            logits = torch.addmm(m.b_out, self.z, m.w_out.T)
            _lib.check(_lib.LIB.pgpb_tbeam_wave_fused(
                self.handle, logits.data_ptr(), self.V, self.lp.data_ptr(), self.V, self.B, self.V, m.blank_id,
                float(self.cfg.lam), int(self.use), k, _lib.ctypes.byref(self.state), self.enc_proj.data_ptr(),
                self.T * m.J, m.J, m.pred_j.data_ptr(), self.z.data_ptr(), _lib.stream_ptr()),
                "pgpb_tbeam_wave_fused")
            return
        else:
            tf = torch.minimum(self.t, (self.lengths - 1).clamp(min=0)).long()
            self.lp.copy_(m.joint_logprobs(self.enc_proj[self.rows, tf], self.hyps.last))
        _lib.check(_lib.LIB.pgpb_tbeam_wave(self.handle, self.lp.data_ptr(), self.V, self.B, self.V, m.blank_id,
                                            float(self.cfg.lam), int(self.use), k, _lib.ctypes.byref(self.state),
                                            _lib.stream_ptr()), "pgpb_tbeam_wave")

    def _frame(self, record=None):
        for k in range(self.cap + 1):
            if record is not None:
                snap = (self.hyps.flags.cpu().numpy(), self.hyps.last.cpu().numpy(), self.t.cpu().numpy())
            self._wave(k)
            if record is not None:
                record.append((self.lp.cpu().numpy().reshape(self.B, self.K, self.V), *snap))

    def _reset(self, enc_proj, lengths):
        torch = self.torch
        B, T = enc_proj.shape[0], enc_proj.shape[1]
        if B != self.B or T > self.T:
            raise ValueError("batch geometry differs from the decoder's")
        self.enc_proj[:, :T].copy_(enc_proj)
        ln = torch.as_tensor(lengths, device=self.dev) if lengths is not None else torch.full((B,), T, device=self.dev)
        _check_lengths(ln, B, T)
        self.lengths.copy_(ln.to(torch.int32))
        self.hyps.reset()
        self.pool.reset()
        self.pool_count.zero_()
        self.trace.reset()
        self.t.zero_()

    def _capture(self):
        torch = self.torch
        s = torch.cuda.Stream(self.dev)
        s.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(s):
            self._frame()
        torch.cuda.current_stream(self.dev).wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._frame()
        self.graph = g

    def run(self, enc_proj, lengths=None, *, record: bool = False):
        """Decode on the device; results stay in the decoder's buffers."""
        if self.use_graph and self.graph is None and not record:
            self._reset(enc_proj, lengths)
            self._capture()
        self._reset(enc_proj, lengths)
        if self.fused:
            self._hidden()  # frame 0, wave 0 (later waves: the fused kernel)
        n_frames = int(self.lengths.max().item()) if self.B else 0
        records = [] if record else None
        for _ in range(n_frames):
            if record:
                self._frame(records)
            elif self.graph is not None:
                self.graph.replay()
            else:
                self._frame()
        self.launches = n_frames * (self.cap + 1)
        return records

    def results(self, vocab=None, want_trace: bool = False) -> list:
        hy, tr = self.hyps.host(), self.trace.host()
        return [_collect(hy, tr, b, self.cfg.lam, vocab, want_trace) for b in range(self.B)]

    def decode(self, enc_proj, lengths=None, *, record: bool = False, vocab=None, want_trace: bool = False):
        records = self.run(enc_proj, lengths, record=record)
        return BeamOutput(self.results(vocab, want_trace), records)


def transducer_beam_batch(model: StatelessTransducerModel, enc, lengths=None, table: ArcTable | None = None,
                          cfg: DecodeConfig | None = None, *, rollback: bool | None = None, vocab=None,
                          want_trace: bool = False) -> list:
    """Batched boosted transducer beam search over enc [B,T,D]: per utterance (best, nbest)."""
    cfg = cfg or DecodeConfig()
    dec = TransducerBeamDecoder(model, table, cfg, enc.shape[0], enc.shape[1], rollback=rollback)
    out = dec.decode(model.project_encoder(enc), lengths, vocab=vocab, want_trace=want_trace)
    return [(nb[0] if nb else None, nb) for nb in out.nbest]


# ---------------------------------------------------------------------------
# AED (config 4)


class TransformerAEDModel:
    """Random-init pre-norm transformer decoder (Canary-style shapes: d=256,
    4 layers, 4 heads, FF 1024) with cross-attention to an encoder memory.

    Step API for beam search over N = B*K slots: `start(memory)` precomputes
    the cross-attention keys/values, `step(tokens, pos)` consumes one token
    per slot at position `pos` (KV-cached self-attention) and returns
    [N, V] f32 log-probs, `reorder(index)` permutes the caches by slot.
    Token id V is the start symbol.
    """

    def __init__(self, vocab_size: int, d_model: int = 256, n_layers: int = 4, n_heads: int = 4, d_ff: int = 1024,
                 max_len: int = 64, seed: int = 0, device="cuda", dtype=None, eos_id: int | None = None,
                 eos_bias: float = 0.0, eos_ramp: float = 0.0):
        torch = _torch()
        g = torch.Generator(device="cpu")
        g.manual_seed(seed)
        dt = dtype or torch.bfloat16
        self.V, self.d, self.L, self.h, self.dff, self.max_len, self.dtype = (vocab_size, d_model, n_layers, n_heads,
                                                                            d_ff, max_len, dt)
        self.dev = torch.device(device)

        def w(*shape, fan_in):
            return (torch.randn(*shape, generator=g) / math.sqrt(fan_in)).to(device=device, dtype=dt)

        d = d_model
        self.emb = w(vocab_size + 1, d, fan_in=1.0)
        self.pos = w(max_len + 1, d, fan_in=1.0) * 0.1
        self.layers = []
        for _ in range(n_layers):
            self.layers.append({
                "wqkv": w(3 * d, d, fan_in=d), "wo": w(d, d, fan_in=d),
                "wq_x": w(d, d, fan_in=d), "wkv_x": w(2 * d, d, fan_in=d), "wo_x": w(d, d, fan_in=d),
                "w1": w(d_ff, d, fan_in=d), "w2": w(d, d_ff, fan_in=d_ff),
            })
        self.w_out = w(vocab_size, d, fan_in=d) * 3.0
        # eos logit offset eos_bias + eos_ramp * pos: sets where synthetic
        # hypotheses end (a random-init decoder otherwise never prefers eos)
        self.eos_id, self.eos_bias, self.eos_ramp = eos_id, float(eos_bias), float(eos_ramp)

    @staticmethod
    def _norm(x):
        import torch.nn.functional as F

        return F.rms_norm(x, (x.shape[-1],))

    def start(self, memory, beam: int):
        """memory [B, Tm, d] -> cross K/V per layer; resets the self-attention caches for B*beam slots."""
        torch = _torch()
        B, Tm, d = memory.shape
        h, dh = self.h, d // self.h
        mem = memory.to(self.dtype)
        same = getattr(self, "N", None) == B * beam and getattr(self, "B", None) == B and \
            self.cross and self.cross[0][0].shape[2] == Tm
        self.B, self.K, self.N = B, beam, B * beam
        # buffers are reused in place when the geometry repeats, so captured
        # decode steps (AEDBeamDecoder graphs) keep valid addresses
        if not same:
            self.cross = []
        for li, lyr in enumerate(self.layers):
            kv = (mem @ lyr["wkv_x"].T).view(B, Tm, 2, h, dh).permute(2, 0, 3, 1, 4)  # [2, B, h, Tm, dh]
            if same:
                self.cross[li][0].copy_(kv[0])
                self.cross[li][1].copy_(kv[1])
            else:
                self.cross.append((kv[0].contiguous(), kv[1].contiguous()))
        if same:
            self.kc.zero_()
            self.vc.zero_()
        else:
            self.kc = torch.zeros((self.L, self.N, h, self.max_len + 1, dh), dtype=self.dtype, device=memory.device)
            self.vc = torch.zeros_like(self.kc)

    def step(self, tokens, pos: int):
        """tokens [N] (start symbol = V) at position pos -> [N, V] f32 log-probs."""
        import torch.nn.functional as F

        torch = _torch()
        N, d, h = self.N, self.d, self.h
        dh = d // h
        x = self.emb[tokens.long()] + self.pos[pos]
        for li, lyr in enumerate(self.layers):
            y = self._norm(x)
            q, k, v = (y @ lyr["wqkv"].T).view(N, 3, h, dh).unbind(1)
            self.kc[li, :, :, pos] = k
            self.vc[li, :, :, pos] = v
            a = F.scaled_dot_product_attention(q.unsqueeze(2), self.kc[li, :, :, :pos + 1], self.vc[li, :, :, :pos + 1])
            x = x + a.reshape(N, d) @ lyr["wo"].T
            y = self._norm(x)
            qx = (y @ lyr["wq_x"].T).view(self.B, self.K, h, dh).transpose(1, 2)  # [B, h, K, dh]
            kx, vx = self.cross[li]
            ax = F.scaled_dot_product_attention(qx, kx, vx)  # [B, h, K, dh]
            x = x + ax.transpose(1, 2).reshape(N, d) @ lyr["wo_x"].T
            y = self._norm(x)
            x = x + F.gelu(y @ lyr["w1"].T) @ lyr["w2"].T
        logits = (self._norm(x) @ self.w_out.T).float()
        if self.eos_id is not None and (self.eos_bias or self.eos_ramp):
            logits[:, self.eos_id] += self.eos_bias + self.eos_ramp * pos
        return torch.log_softmax(logits, dim=-1)

    def reorder(self, index, upto: int):
        """Slot i takes the caches of slot index[i] (positions 0..upto)."""
        self.kc[:, :, :, :upto + 1] = self.kc[:, index, :, :upto + 1]
        self.vc[:, :, :, :upto + 1] = self.vc[:, index, :, :upto + 1]


class AEDBeamDecoder:
    """Batched boosted AED beam search (R10): one decoder step for all B*beam
    slots, then one pgpb_aed_step launch, then the KV-cache reorder."""

    def __init__(self, model: TransformerAEDModel, table: ArcTable | None, cfg: DecodeConfig, batch: int, *,
                 max_len: int, eos: int, device=None, poll: int = 4, use_graph: bool = True):
        torch = _torch()
        self.torch, self.model, self.table, self.cfg = torch, model, table, cfg
        if table is not None and table.vocab_size != model.V:
            raise ValueError(f"step model vocab size {model.V} != table vocab size {table.vocab_size}")
        if max_len < 1:
            raise ValueError(f"max_len must be >= 1, got {max_len}")
        if max_len > model.max_len:
            raise ValueError("max_len exceeds the model's positional table")
        if cfg.beam_size > 32:
            raise ValueError("device beam search supports beam_size <= 32")
        self.B, self.K, self.V, self.max_len, self.eos, self.poll = batch, cfg.beam_size, model.V, max_len, eos, poll
        self.use = _boost_active(table, cfg)
        self.dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.handle = table.device_table(self.dev.index).handle if self.use else None
        row_max = table.device_table(self.dev.index).row_max() if (self.use and cfg.eos_bump_enabled) else None
        self._row_max = row_max
        B, K, d = batch, self.K, self.dev
        self.hyps = _Hyps(torch, B, K, d)
        self.trace = _Trace(torch, B, (max_len + 1) * K + 1, d)
        self.any_active = torch.zeros(1, dtype=torch.int32, device=d)
        self.flag_host = torch.zeros(1, dtype=torch.int32, pin_memory=True)
        self.slot_base = (torch.arange(B, device=d, dtype=torch.int64) * K).unsqueeze(1)
        self.state = _lib.AedState(self.hyps.struct(), self.trace.struct(),
                                   row_max.data_ptr() if row_max is not None else None, self.any_active.data_ptr(),
                                   K, max_len, eos, int(bool(cfg.eos_bump_enabled)), int(bool(cfg.rollback)))
        self.launches = 0
        self.use_graph, self._warm, self.graphs = use_graph, False, {}
        self.pool = torch.cuda.graph_pool_handle() if use_graph else None

    def _step(self, n: int, records=None):
        torch, m = self.torch, self.model
        tokens = torch.where(self.hyps.last < 0, torch.full_like(self.hyps.last, m.V), self.hyps.last).view(-1)
        lp = m.step(tokens, n)
        if records is not None:
            records.append((lp.cpu().numpy().reshape(self.B, self.K, self.V), self.hyps.host(), self.trace.host()))
        self.any_active.zero_()
        _lib.check(_lib.LIB.pgpb_aed_step(self.handle, lp.data_ptr(), self.V, self.B, self.V, float(self.cfg.lam),
                                          int(self.use), _lib.ctypes.byref(self.state), _lib.stream_ptr()),
                   "pgpb_aed_step")
        m.reorder((self.slot_base + self.hyps.parent.long()).view(-1), n)

    def run(self, memory, *, record: bool = False):
        """One batch decode.  With use_graph, the first run is eager (warm-up),
        the second captures every step position as a CUDA graph (one shared
        pool, replayed in capture order) and later runs replay them: a step is
        ~60 small kernels, launch-bound when issued one by one."""
        torch, m = self.torch, self.model
        m.start(memory, self.K)
        self.hyps.reset()
        self.trace.reset()
        records = [] if record else None
        self.launches = 0
        graphs = self.use_graph and not record and self._warm
        for n in range(self.max_len + 1):
            if graphs:
                g = self.graphs.get(n)
                if g is None:
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, pool=self.pool):
                        self._step(n)
                    self.graphs[n] = g
                g.replay()
            else:
                self._step(n, records)
            self.launches += 1
            if (n + 1) % self.poll == 0 or n == self.max_len:
                self.flag_host.copy_(self.any_active, non_blocking=True)
                torch.cuda.current_stream(self.dev).synchronize()
                if int(self.flag_host[0]) == 0:
                    break
        if not record:
            self._warm = True
        return records

    def results(self, vocab=None, want_trace: bool = False) -> list:
        hy, tr = self.hyps.host(), self.trace.host()
        return [_collect(hy, tr, b, self.cfg.lam, vocab, want_trace, eos=self.eos) for b in range(self.B)]

    def decode(self, memory, *, record: bool = False, vocab=None, want_trace: bool = False) -> BeamOutput:
        records = self.run(memory, record=record)
        return BeamOutput(self.results(vocab, want_trace), records)


class AEDGreedyDecoder:
    """Batched boosted greedy AED (aed_beam_boosted at beam 1, R10): per step
    one decoder step for the B utterances (TransformerAEDModel with one slot
    each) and one pgpb_aed_greedy_step launch that fuses the argmax, the
    boosted rerank and the eos bump.  Each step position
    is captured as a CUDA graph on the second run and replayed afterwards."""

    def __init__(self, model: TransformerAEDModel, table: ArcTable | None, cfg: DecodeConfig, batch: int, *,
                 max_len: int, eos: int, device=None, poll: int = 4, use_graph: bool = True):
        torch = _torch()
        self.torch, self.model, self.table, self.cfg = torch, model, table, cfg
        if table is not None and table.vocab_size != model.V:
            raise ValueError(f"step model vocab size {model.V} != table vocab size {table.vocab_size}")
        if max_len < 1:
            raise ValueError(f"max_len must be >= 1, got {max_len}")
        if max_len > model.max_len:
            raise ValueError("max_len exceeds the model's positional table")
        self.B, self.V, self.max_len, self.eos, self.poll = batch, model.V, max_len, eos, poll
        self.use = _boost_active(table, cfg)
        self.dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.handle = table.device_table(self.dev.index).handle if self.use else None
        bump = self.use and cfg.eos_bump_enabled
        dt = table.device_table(self.dev.index) if bump else None
        self._row_max = dt.row_max() if bump else None
        self._final = dt.final_bonus() if bump else None
        B, d = batch, self.dev
        i32, i64, f64 = torch.int32, torch.int64, torch.float64
        self.tree = torch.zeros(B, dtype=i32, device=d)
        self.am = torch.zeros(B, dtype=f64, device=d)
        self.boost = torch.zeros(B, dtype=f64, device=d)
        self.len = torch.zeros(B, dtype=i32, device=d)
        self.ended = torch.zeros(B, dtype=torch.uint8, device=d)
        self.feed = torch.full((B,), model.V, dtype=i64, device=d)
        self.tokens = torch.zeros((B, max_len), dtype=i32, device=d)
        self.deltas = torch.zeros((B, max_len + 1), dtype=f64, device=d)
        self.states = torch.zeros((B, max_len + 1), dtype=i32, device=d)
        self.any_active = torch.zeros(1, dtype=i32, device=d)
        self.flag_host = torch.zeros(1, dtype=i32, pin_memory=True)
        p = lambda x: None if x is None else x.data_ptr()  # noqa: E731
        self.state = _lib.AedGreedyState(p(self.tree), p(self.am), p(self.boost), p(self.len), p(self.ended),
                                         p(self.feed), p(self.tokens), p(self.deltas), p(self.states),
                                         p(self._row_max), p(self._final), p(self.any_active), max_len, eos,
                                         int(bool(cfg.rollback)))
        self.launches = 0
        self.use_graph, self._warm, self.graphs = use_graph, False, {}
        self.pool = torch.cuda.graph_pool_handle() if use_graph else None

    def _reset(self):
        for x in (self.tree, self.am, self.boost, self.len, self.ended):
            x.zero_()
        self.feed.fill_(self.model.V)

    def _step(self, n: int, records=None):
        lp = self.model.step(self.feed, n)
        if records is not None:
            records.append((lp.cpu().numpy(), self.len.cpu().numpy().copy(), self.ended.cpu().numpy().copy()))
        self.any_active.zero_()
        _lib.check(_lib.LIB.pgpb_aed_greedy_step(self.handle, lp.data_ptr(), self.V, self.B, self.V,
                                                 float(self.cfg.lam), int(self.use), _lib.ctypes.byref(self.state),
                                                 _lib.stream_ptr()), "pgpb_aed_greedy_step")

    def run(self, memory, *, record: bool = False):
        torch, m = self.torch, self.model
        m.start(memory, 1)
        self._reset()
        records = [] if record else None
        self.launches = 0
        graphs = self.use_graph and not record and self._warm
        for n in range(self.max_len):
            if graphs:
                g = self.graphs.get(n)
                if g is None:
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, pool=self.pool):
                        self._step(n)
                    self.graphs[n] = g
                g.replay()
            else:
                self._step(n, records)
            self.launches += 1
            if (n + 1) % self.poll == 0 or n + 1 == self.max_len:
                self.flag_host.copy_(self.any_active, non_blocking=True)
                torch.cuda.current_stream(self.dev).synchronize()
                if int(self.flag_host[0]) == 0:
                    break
        if not record:
            self._warm = True
        return records

    def results(self, vocab=None, want_trace: bool = False) -> list[DecodeResult]:
        n = self.len.cpu().numpy()
        ended = self.ended.cpu().numpy()
        tok, dl, st = self.tokens.cpu().numpy(), self.deltas.cpu().numpy(), self.states.cpu().numpy()
        am, bo = self.am.cpu().numpy(), self.boost.cpu().numpy()
        out = []
        for b in range(self.B):
            k = int(n[b])
            tokens = [int(x) for x in tok[b, :k]]
            trace = None
            if want_trace:
                trace = [TraceStep(int(tok[b, i]), float(dl[b, i]), int(st[b, i])) for i in range(k)]
                if ended[b]:
                    trace.append(TraceStep(self.eos, float(dl[b, k]), int(st[b, k])))
            out.append(DecodeResult(tokens, _text(tokens, vocab), float(am[b]), float(bo[b]), trace))
        return out

    def decode(self, memory, *, record: bool = False, vocab=None, want_trace: bool = False):
        records = self.run(memory, record=record)
        return BeamOutput(self.results(vocab, want_trace), records)


# ---------------------------------------------------------------------------
# CTC prefix beam (batched, device resident)


def _logaddexp(a: float, b: float) -> float:  # decoding.py:94-100
    if a == float("-inf"):
        return b
    if b == float("-inf"):
        return a
    m = a if a > b else b
    return m + math.log1p(math.exp(-abs(a - b)))


def ctc_beam_batch(logprobs, lengths=None, table: ArcTable | None = None, cfg: DecodeConfig | None = None, *,
                   blank_id: int, vocab=None, want_trace: bool = False):
    """Boosted CTC prefix beam search (decoding.py:232-343, R8) for a batch:
    one pgpb_ctc_beam launch decodes every frame of every utterance on the
    device (beam <= 32).  logprobs: [B, T, V] float32 (CUDA tensor or
    numpy); lengths: [B] frames or None.  Returns per utterance the
    reference's (best, nbest) pair.  Tokens, boosts and traces are exact; am
    is within an ulp-level difference of the host's logaddexp."""
    torch = _torch()
    cfg = cfg or DecodeConfig()
    lp = logprobs if isinstance(logprobs, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(logprobs, np.float32))
    lp = lp.to(device="cuda", dtype=torch.float32).contiguous()
    if lp.dim() != 3:
        raise ValueError("logprobs must be [B, T, V]")
    B, T, V = lp.shape
    if table is not None and V != table.vocab_size:
        raise ValueError(f"emission vocab size {V} != table vocab size {table.vocab_size}")
    if not 0 <= blank_id < V:
        raise ValueError(f"blank id {blank_id} out of range [0, {V})")
    K = cfg.beam_size
    if K > 32:
        raise ValueError("device CTC beam search supports beam_size <= 32 (use ctc_beam_boosted for wider beams)")
    ln = None
    if lengths is not None:
        ln = torch.as_tensor(np.asarray(lengths) if not isinstance(lengths, torch.Tensor) else lengths)
        from .rnnt import _check_lengths

        _check_lengths(ln, B, T)
        ln = ln.to(device=lp.device, dtype=torch.int32).contiguous()
    o, tr = ctc_beam_device(lp, ln, table, cfg, blank_id)
    if int(o.pop("overflow").item()):
        raise RuntimeError("CTC beam trace overflow")
    h = {k: v.cpu().numpy() for k, v in o.items()}
    t = {k: v.cpu().numpy() for k, v in tr.items()}
    lam = cfg.lam
    if cfg.rollback and _boost_active(table, cfg) and T > 0:  # extension: see DecodeConfig.rollback
        bt = table.device_table(lp.device.index).backoff_total().cpu().numpy()
        h["boost"] = h["boost"] + bt[h["tree"]].astype(np.float64)
    results = []
    for b in range(B):
        out = []
        for r in range(int(h["count"][b])):
            steps = _walk(t, b, int(h["node"][b, r]))
            toks = [s_[0] for s_ in steps]
            am = _logaddexp(float(h["pb"][b, r]), float(h["pnb"][b, r]))
            out.append((toks, am, float(h["boost"][b, r]), steps))
        out.sort(key=lambda x: (-(x[1] + lam * x[2]), -x[1], tuple(x[0])))
        nbest = [DecodeResult(list(tk), _text(tk, vocab), a, bo, [TraceStep(*s_) for s_ in sp] if want_trace else None)
                 for tk, a, bo, sp in out[:K]]
        results.append((nbest[0] if nbest else None, nbest))
    return results


def ctc_beam_device(lp, lengths, table, cfg: DecodeConfig, blank_id: int):
    """The pgpb_ctc_beam launch alone (no host synchronisation except the
    trace-overflow check): lp [B, T, V] float32 CUDA, lengths int32 CUDA [B]
    or None.  Returns (final beams, trace) dicts of device tensors."""
    torch = _torch()
    B, T, V = lp.shape
    K = cfg.beam_size
    ln = lengths
    use = _boost_active(table, cfg)
    dev = lp.device
    nmax = T * K + 1
    f64, i32 = torch.float64, torch.int32
    o = {k: torch.zeros((B, K), dtype=f64, device=dev) for k in ("pb", "pnb", "boost")}
    o.update({k: torch.zeros((B, K), dtype=i32, device=dev) for k in ("tree", "len", "node")})
    o["count"] = torch.zeros(B, dtype=i32, device=dev)
    tr = {k: torch.zeros((B, nmax), dtype=i32, device=dev) for k in ("parent", "token", "state")}
    tr["delta"] = torch.zeros((B, nmax), dtype=f64, device=dev)
    ovf = torch.zeros(1, dtype=i32, device=dev)
    p = lambda x: x.data_ptr()  # noqa: E731
    st = _lib.CtcBeamOut(p(o["pb"]), p(o["pnb"]), p(o["boost"]), p(o["tree"]), p(o["len"]), p(o["node"]),
                         p(o["count"]), p(tr["parent"]), p(tr["token"]), p(tr["state"]), p(tr["delta"]), nmax, p(ovf))
    handle = table.device_table(dev.index).handle if use else None
    _lib.check(_lib.LIB.pgpb_ctc_beam(handle, lp.data_ptr(), B, T, V, None if ln is None else ln.data_ptr(),
                                      int(blank_id), K, float(cfg.lam), int(use), _lib.ctypes.byref(st),
                                      _lib.stream_ptr()), "pgpb_ctc_beam")
    o["overflow"] = ovf
    return o, tr
