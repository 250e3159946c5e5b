"""Device CTC prefix beam: CTA-0 phase timeline, boosted vs unboosted
(needs PGPB_LIB_PATH=.../libpgpb_cbprof.so built with -DPGPB_CB_PROFILE)."""
import ctypes
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
from paper_2508_07014_b200 import _lib  # noqa: E402
from paper_2508_07014_b200.beams import ctc_beam_device  # noqa: E402

f = _lib.LIB.pgpb_debug_cb_profile
f.argtypes = [ctypes.c_void_p, ctypes.c_int]
names = ["carries+wait", "marking", "carried(t0)", "warp-topk+bar", "merge", "winners+end", "-", "dense(t0)", "closure(t0)", "bare-barrier"]
tab, V = bw.table("p20k_v1024")
dev = torch.device("cuda", 0)
for regime, lp, _ in bench._ctc_regimes(64, 200, V, dev, 0):
    if regime not in ("clean", "dense"):
        continue
    lp = lp.contiguous()
    for thr, lam in [(t, l) for t in (1024,) for l in (0.0, 1.0)]:
        _lib.set_tuning("cb.threads", thr)
        cfg = pb.DecodeConfig(lam=lam, beam_size=4)
        ctc_beam_device(lp, None, tab, cfg, 0)
        torch.cuda.synchronize()
        buf = np.zeros(16, np.uint64)
        f(buf.ctypes.data, 1)
        ctc_beam_device(lp, None, tab, cfg, 0)
        torch.cuda.synchronize()
        f(buf.ctypes.data, 1)
        fr = max(int(buf[15]), 1)
        ph = {k: round(int(buf[i]) / fr) for i, k in enumerate(names)}
        print(regime, "threads", thr, "lam", lam, "frames", fr, "cycles/frame", round(sum(int(buf[i]) for i in range(9)) / fr), ph,
              flush=True)
