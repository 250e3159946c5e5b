"""Greedy CTC decode timing sweep (device-timed CUDA graph replays)."""
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import gen_inputs as gi  # noqa: E402

import paper_2508_07014_b200 as pb  # noqa: E402

phrases, V = gi.corpus("p20k_v1024")
ctx = pb.ContextList([pb.Phrase(" ".join(map(str, p)), p) for p in phrases], min_chars=0)
tab = pb.compile_arc_table(pb.compute_fail_links(pb.build_prefix_tree(ctx, pb.TreeParams(), V)))
B, T = int(sys.argv[1]) if len(sys.argv) > 1 else 128, 200
g = torch.Generator(device="cuda")
g.manual_seed(0)
out = {}
for regime in ("dense", "blank3"):
    logits = torch.randn((B, T, V), generator=g, device="cuda") * 2.0
    if regime == "blank3":
        logits[:, torch.arange(T, device="cuda") % 4 != 0, 0] += 10.0
    lp = torch.log_softmax(logits, dim=-1).contiguous()
    for lam in (0.0, 1.0):
        cfg = pb.DecodeConfig(lam=lam)
        o = pb.ctc_greedy_device(lp, None, tab, cfg, 0)
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            for _ in range(10):
                pb.ctc_greedy_device(lp, None, tab, cfg, 0, out=o)
        gr.replay()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        gr.replay()
        e.record()
        torch.cuda.synchronize()
        out[f"{regime}_lam{lam}"] = round(s.elapsed_time(e) / 10 * 1000, 1)
print(json.dumps(out))
