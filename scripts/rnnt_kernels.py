"""Per-kernel device times of one fused RNN-T label iteration, boosted vs
unboosted (torch profiler, eager iterations; config-2 shapes)."""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import gen_inputs as gi  # noqa: E402

import paper_2508_07014_b200 as pb  # noqa: E402
from paper_2508_07014_b200.rnnt import LabelLoopingDecoder, RNNTModel  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

phrases, V = gi.corpus("p20k_v1024")
ctx = pb.ContextList([pb.Phrase(" ".join(map(str, p)), p) for p in phrases], min_chars=0)
tab = pb.compile_arc_table(pb.compute_fail_links(pb.build_prefix_tree(ctx, pb.TreeParams(), V)))
B, T = 128, 200
model = RNNTModel(V, enc_dim=512, pred_dim=640, joint_dim=640, seed=11, blank_bias=10.5)
enc_proj = model.project_encoder(torch.randn((B, T, 512), device="cuda", generator=torch.Generator(device="cuda").manual_seed(0)))
for lam in (0.0, 1.0):
    dec = LabelLoopingDecoder(model, tab, pb.DecodeConfig(lam=lam), B, T, use_graph=False)
    dec._reset(enc_proj, None)
    for _ in range(20):
        dec._iteration()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(50):
            dec._iteration()
        torch.cuda.synchronize()
    print("lam", lam)
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12))
