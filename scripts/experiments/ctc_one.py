"""One boosted fused-CTC call per regime (for ncu captures)."""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "scripts"))
import ctc_regimes as cr  # noqa: E402

import paper_2508_07014_b200 as pb  # noqa: E402

regime = sys.argv[1] if len(sys.argv) > 1 else "clean"
lam = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
tab, V = cr.table()
lp = cr.regimes(128, 200, V, torch.device("cuda"))[regime]
for _ in range(3):
    o = pb.ctc_greedy_device(lp, None, tab, pb.DecodeConfig(lam=lam), 0)
torch.cuda.synchronize()
