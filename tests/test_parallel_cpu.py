"""Multi-process data-parallel plumbing on CPU (gloo, world size 2).

Decoding itself needs the GPU; these tests cover the host side of the
multi-GPU path: sharding, table replication by broadcast and the single
all-gather of padded hypotheses, which must reproduce the single-process
result list exactly.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _fake_results(n, seed=0):
    from paper_2508_07014_b200.decoding import DecodeResult, TraceStep

    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        k = int(rng.integers(0, 9))
        toks = [int(x) for x in rng.integers(1, 50, size=k)]
        tr = [TraceStep(t, float(rng.normal()), int(rng.integers(0, 99))) for t in toks]
        out.append(DecodeResult(toks, "", float(rng.normal()), float(sum(s.boost for s in tr)), tr))
    return out


def _worker(rank, world, port, n, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import gen_inputs as gi
        from conftest import product_table

        from paper_2508_07014_b200.parallel import all_gather_results, broadcast_table, shard_range

        # table replication: rank 0 builds, everyone receives identical arrays
        tab = product_table(gi.corpus("p100_v1024")[0], 1024) if rank == 0 else None
        tab = broadcast_table(tab, src=0)
        sig = [int(tab.num_states), int(tab.num_arcs), float(tab.arc_weight.sum()), int(tab.backoff_to.sum())]
        # sharded "decode" + one all-gather
        allres = _fake_results(n, seed=3)
        lo, hi = shard_range(n, world, rank)
        got = all_gather_results(allres[lo:hi], n, with_trace=True)
        q.put((rank, sig, [(r.tokens, r.am_score, r.boost_score, [(s.token, s.boost, s.state) for s in r.trace])
                           for r in got]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [7, 8, 1])
def test_gloo_world2_shard_gather_equals_single_process(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    exp = [(r.tokens, r.am_score, r.boost_score, [(s.token, s.boost, s.state) for s in r.trace])
           for r in _fake_results(n, seed=3)]
    sigs = {tuple(o[1]) for o in outs}
    assert len(sigs) == 1
    for _, _, got in outs:
        assert got == exp


def test_shard_range_covers_everything():
    from paper_2508_07014_b200.parallel import shard_range

    for n in (0, 1, 5, 8192):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                lo, hi = shard_range(n, world, r)
                seen.extend(range(lo, hi))
            assert seen == list(range(n))
