"""Chained advance (pgpb_advance_steps) device time vs column parts P and
batch, graph of back-to-back launches over >= 256 MiB of outputs."""
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
peak = 6454.9
R, steps = int(sys.argv[1]) if len(sys.argv) > 1 else 8, 20
rng = np.random.default_rng(1)
for B in ((128, 1024, 8192, 65536) if R == 1 else (1024, 8192, 65536)):
    st = torch.from_numpy(rng.integers(0, tab.num_states, size=(steps, B)).astype(np.int32)).cuda()
    tk = torch.from_numpy(rng.integers(0, V, size=(R, B)).astype(np.int32)).cuda()
    per = R * B * V * 8
    ring = max(2, min(steps, -(-256 * 2**20 // per)))
    outs = [(torch.empty((R, B, V), dtype=torch.float32, device="cuda"),
             torch.empty((R, B, V), dtype=torch.int32, device="cuda")) for _ in range(ring)]
    for P in ((-1, 0, 2, 4) if R == 1 else (0, 1, 2, 4, 8)):
        def step(i):
            s, n = outs[i % ring]
            if P < 0:  # the single-advance kernel (pgpb_advance)
                _lib.check(_lib.LIB.pgpb_advance(dt.handle, st[i].data_ptr(), B, s.data_ptr(), n.data_ptr(),
                                                 _lib.stream_ptr()))
                return
            _lib.check(_lib.LIB.pgpb_advance_steps(dt.handle, st[i].data_ptr(), tk.data_ptr() if R > 1 else None, R,
                                                   B, s.data_ptr(), n.data_ptr(), None, None, P, _lib.stream_ptr()))
        for i in range(3):
            step(i)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(steps):
                step(i)
        g.replay()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b) / steps)
        gbs = R * (B * V * 8 + B * 4) / (best / 1e3) / 1e9
        print(f"R={R} B={B} P={'v6' if P < 0 else (P or 'auto')} {best * 1e3:.1f} us/launch {gbs:.0f} GB/s {gbs / peak:.3f}", flush=True)
    del outs
    torch.cuda.empty_cache()
