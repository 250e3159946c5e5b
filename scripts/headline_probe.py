"""Why the headline replay (one graph of K launches, per-launch state and
token batches) reads lower than the sweep (best of 3 replays, one token
batch): vary the number of distinct input batches, K and the output ring."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import bench_workloads as bw  # noqa: E402

from paper_2508_07014_b200 import _lib  # noqa: E402

tab, V = bw.table("p20k_v1024")
dt = tab.device_table(0)
B = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
R = int(sys.argv[2]) if len(sys.argv) > 2 else 8
PARTS = int(sys.argv[3]) if len(sys.argv) > 3 else 0
LAYOUTS = [int(x) for x in sys.argv[4].split(",")] if len(sys.argv) > 4 else [0, 3]
rng = np.random.default_rng(1000)
big = B * R > 8192 * 8
cases = [(n_in, 8 if big else 50, 2, cm) for cm in LAYOUTS for n_in in ((8 if big else 50), 1)]
for n_in, K, ring, cm in cases:
    _lib.set_tuning("adv.compact", cm)
    st = torch.from_numpy(rng.integers(0, tab.num_states, size=(n_in, B)).astype(np.int32)).cuda()
    tk = torch.from_numpy(rng.integers(0, V, size=(n_in, R, B)).astype(np.int32)).cuda()
    outs = [(torch.empty((R, B, V), dtype=torch.float32, device="cuda"),
             torch.empty((R, B, V), dtype=torch.int32, device="cuda")) for _ in range(ring)]

    def step(i):
        s, n = outs[i % ring]
        _lib.check(_lib.LIB.pgpb_advance_steps(dt.handle, st[i % n_in].data_ptr(), tk[i % n_in].data_ptr(), R, B,
                                               s.data_ptr(), n.data_ptr(), None, None, 0, _lib.stream_ptr()))
    for i in range(3):
        step(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(K):
            step(i)
    ts = []
    for _ in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / K)
    frac = [round(R * (B * V * 8 + B * 4) / (t / 1e3) / 1e9 / 6454.9, 3) for t in ts]
    print(f"B={B} R={R} P={PARTS} n_in={n_in} layout={cm} frac {frac}", flush=True)
    del outs, g
    torch.cuda.empty_cache()
