"""Config-2 RNN-T greedy (label looping) boosted vs unboosted, repeated, to
separate box noise from a regression."""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import bench  # noqa: E402
import bench_workloads as bw  # noqa: E402

tab, V = bw.table("p20k_v1024")
for i in range(4):
    r = bench.bench_rnnt(tab, V, torch.device("cuda", 0), 0, 1)
    print(i, "unboosted", round(r["unboosted"]["ms"], 3), "boosted", round(r["boosted"]["ms"], 3), "overhead",
          round(r["overhead"], 4), flush=True)
