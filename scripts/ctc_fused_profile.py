"""Counters of the fused CTC kernel (needs PGPB_LIB_PATH=.../libpgpb_prof.so,
built by scripts/build_prof_lib.sh)."""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "scripts"))
import ctc_regimes as cr  # noqa: E402

import paper_2508_07014_b200 as pb  # noqa: E402
from paper_2508_07014_b200 import _lib  # noqa: E402

f = _lib.LIB.pgpb_debug_ctc_fused_profile
f.argtypes = [ctypes.c_void_p, ctypes.c_int]
tab, V = cr.table()
B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
T = int(sys.argv[2]) if len(sys.argv) > 2 else 200
names = ["fixup_rounds", "r0_steps", "fix_steps", "warp_dec", "rescans", "cyc_prod", "cyc_r0", "cyc_fix", "cyc_tail",
         "segments", "gathers", "lane_dec_n", "lane_dec_cyc", "am_sum_cyc", "warp_dec_n", "warp_dec_cyc"]
for name, lp in cr.regimes(B, T, V, torch.device("cuda")).items():
    for lam in (0.0, 1.0):
        cfg = pb.DecodeConfig(lam=lam)
        o = pb.ctc_greedy_device(lp, None, tab, cfg, 0)
        torch.cuda.synchronize()
        buf = np.zeros(256, np.uint64)
        f(buf.ctypes.data, 1)
        o = pb.ctc_greedy_device(lp, None, tab, cfg, 0)
        torch.cuda.synchronize()
        f(buf.ctypes.data, 1)
        print(name, lam, {k: int(buf[i]) for i, k in enumerate(names)}, "emitted/utt",
              float(o.num_out.double().mean()), flush=True)
        if lam:
            print("  steps(cyc):", [int(v) for v in buf[16:16 + 60]])
            print("  emit/need :", [int(v) for v in buf[128:128 + 60]])
            print("  timeline: staged", int(buf[200]), "accountant", int(buf[201]), "guess", [int(v) for v in buf[210:214]],
                  "round0", [int(v) for v in buf[220:224]], "walk done", int(buf[230]), "boost sum", int(buf[231]),
                  "tail end", int(buf[8]))
