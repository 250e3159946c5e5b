"""Per-phase cycles of the transducer wave kernel at the config-3 shape
(needs PGPB_LIB_PATH=.../libpgpb_tbprof.so built with -DPGPB_TBEAM_PROFILE:
scripts/experiments/build_prof_lib.sh with PROF_FLAG=-DPGPB_TBEAM_PROFILE)."""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import bench_workloads as bw  # noqa: E402

import paper_2508_07014_b200 as pb  # noqa: E402
from paper_2508_07014_b200 import _lib  # noqa: E402
from paper_2508_07014_b200.beams import TransducerBeamDecoder  # noqa: E402

f = _lib.LIB.pgpb_debug_tbeam_profile
f.argtypes = [ctypes.c_void_p, ctypes.c_int]
model, tab, enc = bw.config3(torch.device("cuda", 0))
c = bw.C3
for lam in (0.0, 1.0):
    dec = TransducerBeamDecoder(model, tab, pb.DecodeConfig(lam=lam, beam_size=4, max_symbols_per_frame=5), c["B"],
                                c["T"], use_graph=False)
    dec.run(enc)
    torch.cuda.synchronize()
    buf = np.zeros(16, np.uint64)
    f(buf.ctypes.data, 1)
    dec.run(enc)
    torch.cuda.synchronize()
    f(buf.ctypes.data, 1)
    waves = c["T"] * 6
    names = ["stage", "merge", "mark", "scan", "topk", "winners"]
    print("lam", lam, {n: round(int(buf[i]) / waves / 1.965e3, 2) for i, n in enumerate(names)}, "us per wave (CTA 0)")
    wn = ["w:to-expansion", "w:blobs", "w:closure", "w:scan", "w:topk"]
    print("  thread 32:", {n: round(int(buf[7 + i]) / waves / 1.965e3, 2) for i, n in enumerate(wn)})
