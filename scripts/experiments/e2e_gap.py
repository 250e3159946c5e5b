"""Where the e2e step's time goes: get_scores_batch(numpy) wall time vs the
host successor gather vs a bare pinned D2H of the same bytes (8192 x 1024)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import bench  # noqa: E402

import paper_2508_07014_b200 as pb  # noqa: E402

tab, phrases, V = bench.build_table()
B = 8192
rng = np.random.default_rng(0)
st = rng.integers(0, tab.num_states, size=B).astype(np.int32)
tok = rng.integers(0, V, size=(40, B)).astype(np.int32)
ar = np.arange(B)
for _ in range(5):
    r = pb.get_scores_batch(tab, st)
t_call, t_gather = [], []
s = st
for k in range(32):
    t0 = time.perf_counter()
    r = pb.get_scores_batch(tab, s)
    t1 = time.perf_counter()
    s = r.next_states[ar, tok[k]]
    t2 = time.perf_counter()
    t_call.append(t1 - t0)
    t_gather.append(t2 - t1)
d = torch.empty((B, V), dtype=torch.float32, device="cuda")
h = torch.empty((B, V), dtype=torch.float32, pin_memory=True)
for _ in range(3):
    h.copy_(d)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    h.copy_(d, non_blocking=True)
torch.cuda.synchronize()
t_copy = (time.perf_counter() - t0) / 10
print("call ms median", round(1e3 * float(np.median(t_call)), 3), "gather ms median", round(1e3 * float(np.median(t_gather)), 3),
      "bare 32MB pinned D2H ms", round(1e3 * t_copy, 3), "-> two copies", round(2e3 * t_copy, 3))
# call pieces
import paper_2508_07014_b200.table as T  # noqa: E402
t0 = time.perf_counter()
for _ in range(20):
    a, b_ = T._host_out(B, V)
t1 = time.perf_counter()
print("_host_out ms", round(1e3 * (t1 - t0) / 20, 3))
