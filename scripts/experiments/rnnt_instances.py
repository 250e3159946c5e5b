"""Config-2 label looping: time several decoder instances per configuration
(instances differ by their buffers / captured graphs, not their work)."""
import statistics
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import bench_workloads as bw  # noqa: E402

import paper_2508_07014_b200 as pb  # noqa: E402
from paper_2508_07014_b200.rnnt import LabelLoopingDecoder  # noqa: E402

dev = torch.device("cuda", 0)
c = bw.C2
model, tab, enc = bw.config2(dev, 0)
for lam in (0.0, 1.0, 0.0, 1.0):
    decs = [LabelLoopingDecoder(model, tab, pb.DecodeConfig(lam=lam), c["B"], c["T"], use_graph=True) for _ in range(3)]
    res = []
    for d in decs:
        d.decode(enc)
        ts = []
        for _ in range(3):
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            d.decode(enc)
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        res.append(round(statistics.median(ts), 3))
    print("lam", lam, "instances ms", res, flush=True)
    del decs
    torch.cuda.empty_cache()
