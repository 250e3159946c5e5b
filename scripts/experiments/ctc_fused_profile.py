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
            print("  timeline (CTA 0, cycles since entry): prologue", int(buf[200]), "wait released", int(buf[201]),
                  "staged", int(buf[202]), "mode", int(buf[203]), "guessed", int(buf[204]), "round0", int(buf[205]),
                  "walk done", int(buf[206]), "sums", int(buf[207]), "end", int(buf[208]), "scanback", int(buf[212]), "rt1 issued", int(buf[213]), "rt1 used", int(buf[214]), "rt2 lanes", int(buf[22]))
            names2 = {0: "none", 1: "fast", 3: "semi", 5: "root", 8: "scan", 9: "fast>scan", 11: "semi>scan"}
            print("  lane paths (all CTAs):", {f"{names2.get(k, k)}:{'ok' if r else 'fail'}": int(buf[160 + 2 * k + r])
                                               for k in range(16) for r in (0, 1) if buf[160 + 2 * k + r]})
            print("  warp decisions", int(buf[192]), "rescans", int(buf[193]), "round0 per warp: max", int(buf[194]),
                  "mean", int(buf[195]) / max(1, int(buf[196])))
            print("  2nd utterance (entry = start - 5000):", [int(v) for v in buf[220:235]])
            print("  latency: top", int(buf[240]), "blob", int(buf[241]), "top again", int(buf[242]), "bitmap", int(buf[243]),
                  "| at the end: blob", int(buf[244]), "bitmap", int(buf[245]))
