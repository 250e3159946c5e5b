"""One device CTC prefix beam launch (64 x 200 clean, beam 4), lam = argv[1]; for ncu."""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import bench  # noqa: E402
import bench_workloads as bw  # noqa: E402

import paper_2508_07014_b200 as pb  # noqa: E402
from paper_2508_07014_b200.beams import ctc_beam_device  # noqa: E402

lam = float(sys.argv[1])
tab, V = bw.table("p20k_v1024")
for regime, lp, _ in bench._ctc_regimes(64, 200, V, torch.device("cuda", 0), 0):
    if regime == "clean":
        ctc_beam_device(lp.contiguous(), None, tab, pb.DecodeConfig(lam=lam, beam_size=4), 0)
        torch.cuda.synchronize()
print("ok")
