"""Device CTC prefix beam: advance blobs (beam.blobs 0) against closure
records + bitmap marking (1), per bench regime."""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import bench  # noqa: E402
import bench_workloads as bw  # noqa: E402

from paper_2508_07014_b200 import _lib  # noqa: E402

tab, V = bw.table("p20k_v1024")
for mode in (1, 0, 1, 0):
    _lib.set_tuning("beam.blobs", mode)
    r = bench.bench_ctc_beam(tab, V, torch.device("cuda", 0), 0, 1)
    for k, v in r.items():
        if isinstance(v, dict) and "overhead" in v:
            print("blobs" if mode == 0 else "records", k, "unboosted", round(v["unboosted"]["ms"], 4), "boosted",
                  round(v["boosted"]["ms"], 4), "overhead", round(v["overhead"], 4), flush=True)
_lib.set_tuning("beam.blobs", 0)
