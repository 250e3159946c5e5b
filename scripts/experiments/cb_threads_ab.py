"""Device CTC prefix beam: CTA size (tuning key cb.threads) A/B, bench regimes."""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import bench  # noqa: E402
import bench_workloads as bw  # noqa: E402

from paper_2508_07014_b200 import _lib  # noqa: E402

tab, V = bw.table("p20k_v1024")
import os  # noqa: E402

thr_list = [int(x) for x in sys.argv[1:]] or [1024, 512, 256]
scores = [int(x) for x in os.environ.get("CB_SCORES", "0").split(",")]
for rep in range(2):
    for thr, sc in [(t, c) for t in thr_list for c in scores]:
        _lib.set_tuning("cb.threads", thr)
        if "CB_SCORES" in os.environ:
            _lib.set_tuning(os.environ.get("CB_KEY", "cb.scores"), sc)  # only in builds that have the key
        r = bench.bench_ctc_beam(tab, V, torch.device("cuda", 0), 0, 1)
        for k, v in r.items():
            if isinstance(v, dict) and "overhead" in v:
                print("threads", thr, "scores", sc, k, "unboosted", round(v["unboosted"]["ms"], 4), "boosted",
                      round(v["boosted"]["ms"], 4), "overhead", round(v["overhead"], 4), flush=True)
_lib.set_tuning("cb.threads", 0)
