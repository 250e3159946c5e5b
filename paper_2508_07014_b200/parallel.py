"""Data-parallel GPU-PB: utterances sharded over ranks, one all-gather at the end.

One process per GPU (torchrun), `torch.distributed` for the plumbing:

* the compiled table is replicated: every rank can build it
  deterministically, or rank 0 builds it and `broadcast_table` ships the
  GPB1 bytes (table.py:16-29) — ~5 MB at 20K phrases;
* `shard_range` gives each rank a contiguous block of ceil(N / world)
  utterances; decoding is independent per utterance, so
  there is no per-step communication;
* `all_gather_results` packs each rank's DecodeResults into fixed-size
  padded tensors (tokens, trace deltas/states, lengths, am, boost) and runs
  ONE all_gather_into_tensor per field (NCCL over NVLink on GPUs, gloo on
  CPU) — the only collective on the path.
"""

from __future__ import annotations

import math
import tempfile
from pathlib import Path

import numpy as np

from .decoding import DecodeResult, TraceStep


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) of utterances owned by `rank`: contiguous blocks of ceil(n/world)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    per = math.ceil(n / world) if n else 0
    lo = min(n, rank * per)
    return lo, min(n, lo + per)


def _dist():
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        raise RuntimeError("torch.distributed is not initialised")
    return dist


def _device_for(group=None):
    import torch

    dist = _dist()
    backend = dist.get_backend(group)
    if backend == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def broadcast_table(table, src: int = 0, group=None):
    """Replicate an ArcTable from rank `src` to every rank (GPB1 bytes)."""
    import torch

    from .table import load_table, save_table

    dist = _dist()
    dev = _device_for(group)
    rank = dist.get_rank(group)
    if rank == src:
        with tempfile.TemporaryDirectory() as d:
            p = Path(d) / "t.gpb"
            save_table(table, p)
            blob = p.read_bytes()
        n = torch.tensor([len(blob)], dtype=torch.int64, device=dev)
    else:
        n = torch.zeros(1, dtype=torch.int64, device=dev)
    dist.broadcast(n, src, group=group)
    data = torch.empty(int(n.item()), dtype=torch.uint8, device=dev)
    if rank == src:
        data.copy_(torch.frombuffer(bytearray(blob), dtype=torch.uint8))
    dist.broadcast(data, src, group=group)
    if rank == src:
        return table
    with tempfile.TemporaryDirectory() as d:
        p = Path(d) / "t.gpb"
        p.write_bytes(data.cpu().numpy().tobytes())
        return load_table(p)


def pack_results(results: list[DecodeResult], rows: int, lmax: int, with_trace: bool):
    """Fixed-size host arrays for `rows` slots (missing rows have length -1)."""
    tok = np.zeros((rows, lmax), np.int32)
    dl = np.zeros((rows, lmax), np.float64)
    st = np.zeros((rows, lmax), np.int32)
    ln = np.full(rows, -1, np.int32)
    am = np.zeros(rows, np.float64)
    bo = np.zeros(rows, np.float64)
    for i, r in enumerate(results):
        k = len(r.tokens)
        if k > lmax:
            raise ValueError(f"hypothesis of {k} tokens exceeds lmax={lmax}")
        ln[i] = k
        tok[i, :k] = r.tokens
        am[i] = r.am_score
        bo[i] = r.boost_score
        if with_trace and r.trace is not None:
            dl[i, :k] = [s.boost for s in r.trace]
            st[i, :k] = [s.state for s in r.trace]
    return {"tokens": tok, "deltas": dl, "states": st, "lengths": ln, "am": am, "boost": bo}


def unpack_results(packed, vocab=None, with_trace: bool = False) -> list[DecodeResult]:
    from .decoding import _text

    out = []
    for i in range(packed["lengths"].shape[0]):
        k = int(packed["lengths"][i])
        if k < 0:
            continue
        toks = [int(x) for x in packed["tokens"][i, :k]]
        trace = [TraceStep(int(t), float(d), int(s)) for t, d, s in
                 zip(packed["tokens"][i, :k], packed["deltas"][i, :k], packed["states"][i, :k])] if with_trace else None
        out.append(DecodeResult(toks, _text(toks, vocab), float(packed["am"][i]), float(packed["boost"][i]), trace))
    return out


def all_gather_results(local: list[DecodeResult], n_total: int, *, lmax: int | None = None, vocab=None,
                       with_trace: bool = False, group=None) -> list[DecodeResult]:
    """Gather every rank's shard of results, in global utterance order."""
    import torch

    dist = _dist()
    world = dist.get_world_size(group)
    dev = _device_for(group)
    per = math.ceil(n_total / world) if n_total else 0
    if lmax is None:  # agree on the longest hypothesis
        m = torch.tensor([max((len(r.tokens) for r in local), default=0)], dtype=torch.int64, device=dev)
        dist.all_reduce(m, op=dist.ReduceOp.MAX, group=group)
        lmax = max(1, int(m.item()))
    packed = pack_results(local, per, lmax, with_trace)
    gathered = {}
    for name, arr in packed.items():
        src = torch.from_numpy(np.ascontiguousarray(arr)).to(dev)
        dst = torch.empty((world * src.shape[0],) + tuple(src.shape[1:]), dtype=src.dtype, device=dev)
        dist.all_gather_into_tensor(dst, src, group=group)
        gathered[name] = dst.cpu().numpy()
    return unpack_results(gathered, vocab, with_trace)[:n_total]
