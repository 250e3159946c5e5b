"""Config 3 device transducer beam: advance blobs (beam.blobs 0) against
closure records + bitmap marking (1), boosted and unboosted batch time."""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import bench_workloads as bw  # noqa: E402

import paper_2508_07014_b200 as pb  # noqa: E402
from paper_2508_07014_b200 import _lib  # noqa: E402
from paper_2508_07014_b200.beams import TransducerBeamDecoder  # noqa: E402

dev = torch.device("cuda", 0)
model, tab, enc = bw.config3(dev)
c = bw.C3
res = {}
for mode in (1, 0, 1, 0):
    _lib.set_tuning("beam.blobs", mode)
    for lam in (0.0, 1.0):
        dec = TransducerBeamDecoder(model, tab, pb.DecodeConfig(lam=lam, beam_size=4, max_symbols_per_frame=5), c["B"],
                                    c["T"])
        dec.run(enc)
        dec.run(enc)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        dec.run(enc)
        e.record()
        torch.cuda.synchronize()
        res.setdefault((mode, lam), []).append(s.elapsed_time(e))
_lib.set_tuning("beam.blobs", 0)
for (mode, lam), v in sorted(res.items()):
    print("blobs" if mode == 0 else "records", "lam", lam, "ms", [round(x, 2) for x in v], flush=True)
