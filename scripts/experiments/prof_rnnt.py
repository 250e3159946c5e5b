import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import gen_inputs as gi  # noqa: E402

import paper_2508_07014_b200 as pb  # noqa: E402
from paper_2508_07014_b200.rnnt import LabelLoopingDecoder, RNNTModel  # noqa: E402

phrases, V = gi.corpus("p20k_v1024")
ctx = pb.ContextList([pb.Phrase(" ".join(map(str, p)), p) for p in phrases], min_chars=0)
tab = pb.compile_arc_table(pb.compute_fail_links(pb.build_prefix_tree(ctx, pb.TreeParams(), V)))
B, T = 128, 200
for bias in (8.0, 10.0, 10.5, 11.0, 12.0):
    model = RNNTModel(V, enc_dim=512, pred_dim=640, joint_dim=640, seed=11, blank_bias=bias)
    enc_proj = model.project_encoder(torch.randn((B, T, 512), device="cuda"))
    dec = LabelLoopingDecoder(model, tab, pb.DecodeConfig(lam=1.0), B, T, use_graph=True)
    o = dec.decode(enc_proj)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    o = dec.decode(enc_proj)
    e.record()
    torch.cuda.synchronize()
    print(f"bias {bias}: iters {o.iterations} emitted/utt {o.num_out.float().mean().item():.1f} ms {s.elapsed_time(e):.2f} "
          f"us/iter {1000 * s.elapsed_time(e) / o.iterations:.1f}")
model = RNNTModel(V, enc_dim=512, pred_dim=640, joint_dim=640, seed=11, blank_bias=12.0)
enc_proj = model.project_encoder(torch.randn((B, T, 512), device="cuda"))
dec = LabelLoopingDecoder(model, tab, pb.DecodeConfig(lam=1.0), B, T, use_graph=False)
dec._reset(enc_proj, None)
for _ in range(3):
    dec._iteration()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(20):
        dec._iteration()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25))
