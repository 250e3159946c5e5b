"""Device CTC prefix beam (bench.py's decode_ctc_beam leg): boosted vs
unboosted batch time per regime."""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import bench  # noqa: E402
import bench_workloads as bw  # noqa: E402

tab, V = bw.table("p20k_v1024")
r = bench.bench_ctc_beam(tab, V, torch.device("cuda", 0), 0, 1)
for k, v in r.items():
    if isinstance(v, dict) and "overhead" in v:
        print(k, "unboosted", round(v["unboosted"]["ms"], 4), "boosted", round(v["boosted"]["ms"], 4), "overhead",
              round(v["overhead"], 4), flush=True)
