"""Advance-kernel variant sweep (device-timed, ring of outputs > L2) + write-BW baselines."""
import json
import os
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import gen_inputs as gi  # noqa: E402

import paper_2508_07014_b200 as pb  # noqa: E402
from paper_2508_07014_b200 import _lib  # noqa: E402

corpus = sys.argv[1] if len(sys.argv) > 1 else "p20k_v1024"
batches = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "8192").split(",")]
phrases, V = gi.corpus(corpus)
ctx = pb.ContextList([pb.Phrase(" ".join(map(str, p)), p) for p in phrases], min_chars=0)
tab = pb.compile_arc_table(pb.compute_fail_links(pb.build_prefix_tree(ctx, pb.TreeParams(), V)))
h = tab.device_table().handle
rng = np.random.default_rng(0)
res = {"variant": os.environ.get("PGPB_ADVANCE_VARIANT", "default"), "corpus": corpus, "rows": []}


def timeit(fn, n_ring, iters=40, warm=5):
    """Per-launch time from a CUDA graph of `iters` back-to-back launches
    (host submission cost excluded), median over 5 replays."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for i in range(warm):
            fn(i)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(iters):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / iters)
    return statistics.median(ts), statistics.mean(ts)


for B in batches:
    ring = max(2, min(16, (512 << 20) // (B * V * 8) + 1))
    st = [torch.from_numpy(rng.integers(0, tab.num_states, size=B).astype(np.int32)).cuda() for _ in range(4)]
    outs = [(torch.empty((B, V), device="cuda"), torch.empty((B, V), dtype=torch.int32, device="cuda")) for _ in range(ring)]

    def step(i):
        s, n = outs[i % ring]
        _lib.check(_lib.LIB.pgpb_advance(h, st[i % 4].data_ptr(), B, s.data_ptr(), n.data_ptr(), _lib.stream_ptr()))

    med, mean = timeit(step, ring)
    byt = B * V * 8 + B * 4
    row = {"B": B, "ring": ring, "ms_med": med, "ms_mean": mean, "GBps_med": byt / med / 1e6, "GBps_mean": byt / mean / 1e6}
    # write-only baseline on the same bytes
    fl = [torch.empty(B * V * 2, device="cuda") for _ in range(ring)]
    m2, _ = timeit(lambda i: fl[i % ring].fill_(1.0), ring)
    row["fill_GBps"] = B * V * 8 / m2 / 1e6
    # copy baseline (read+write) same output bytes
    src = torch.empty(B * V * 2, device="cuda")
    m3, _ = timeit(lambda i: fl[i % ring].copy_(src), ring)
    row["copy_GBps_rw"] = 2 * B * V * 8 / m3 / 1e6
    # correctness vs oracle on a few rows
    from oracle import oracle as orc
    s, n = outs[39 % ring]
    sts = st[39 % 4].cpu().numpy()[:64]
    sc, nx = orc.score_batch(tab, sts)
    row["exact"] = bool(np.array_equal(s[:64].cpu().numpy().view(np.uint32), sc.view(np.uint32)) and np.array_equal(n[:64].cpu().numpy(), nx))
    res["rows"].append(row)
    del outs, fl
    torch.cuda.empty_cache()
print(json.dumps(res))
