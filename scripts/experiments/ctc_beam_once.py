"""One device CTC prefix-beam launch at the bench shape (64 x 200, beam 4,
clean regime) for an ncu capture: argv[1] = lam."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import bench  # noqa: E402
import bench_workloads as bw  # noqa: E402

import paper_2508_07014_b200 as pb  # noqa: E402
from paper_2508_07014_b200.beams import ctc_beam_device  # noqa: E402

tab, V = bw.table("p20k_v1024")
dev = torch.device("cuda", 0)
lam = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
for regime, lp, lens in bench._ctc_regimes(64, 200, V, dev, 0):
    lp = lp.contiguous()
    for _ in range(3):
        ctc_beam_device(lp, None, tab, pb.DecodeConfig(lam=lam, beam_size=4), 0)
    torch.cuda.synchronize()
    break
print("ok")
