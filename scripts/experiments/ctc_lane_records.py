import ctypes, sys
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, "scripts"); sys.path.insert(0, ".")
import ctc_regimes as cr, paper_2508_07014_b200 as pb
from paper_2508_07014_b200 import _lib
f = _lib.LIB.pgpb_debug_ctc_lane_records; f.argtypes = [ctypes.c_void_p, ctypes.c_int]
tab, V = cr.table()
lp = cr.regimes(128, 200, V, torch.device("cuda"))["clean"]
cfg = pb.DecodeConfig(lam=1.0)
pb.ctc_greedy_device(lp, None, tab, cfg, 0); torch.cuda.synchronize()
buf = np.zeros((256, 4), np.int64); f(buf.ctypes.data, 1)
pb.ctc_greedy_device(lp, None, tab, cfg, 0); torch.cuda.synchronize()
f(buf.ctypes.data, 1)
rows = [r for r in buf if r[0] > 0]
rows.sort(key=lambda r: -r[0])
print("n", len(rows))
for r in rows[:25]: print(list(r))
print("path counts", {p: sum(1 for r in rows if r[2] == p) for p in set(int(r[2]) for r in rows)})
