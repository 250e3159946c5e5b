"""Phase-B checkpoint profile (needs PGPB_LIB_PATH=.../libpgpb_prof.so)."""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import gen_inputs as gi  # noqa: E402

import paper_2508_07014_b200 as pb  # noqa: E402
from paper_2508_07014_b200 import _lib  # noqa: E402

f = _lib.LIB.pgpb_debug_seq_profile
f.argtypes = [ctypes.c_void_p, ctypes.c_int]
phrases, V = gi.corpus("p20k_v1024")
ctx = pb.ContextList([pb.Phrase(" ".join(map(str, p)), p) for p in phrases], min_chars=0)
tab = pb.compile_arc_table(pb.compute_fail_links(pb.build_prefix_tree(ctx, pb.TreeParams(), V)))
for regime in ("dense", "blank3"):
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    logits = torch.randn((128, 200, V), generator=g, device="cuda") * 2.0
    if regime == "blank3":
        logits[:, torch.arange(200, device="cuda") % 4 != 0, 0] += 10.0
    lp = torch.log_softmax(logits, dim=-1).contiguous()
    o = pb.ctc_greedy_device(lp, None, tab, pb.DecodeConfig(lam=1.0), 0)
    torch.cuda.synchronize()
    buf = np.zeros(16, np.uint64)
    f(buf.ctypes.data, 1)
    o = pb.ctc_greedy_device(lp, None, tab, pb.DecodeConfig(lam=1.0), 0)
    torch.cuda.synchronize()
    f(buf.ctypes.data, 1)
    n = int(o.num_out[0].item())
    names = ["nonemit", "ring_get", "pred_blob", "rerank", "ring_refill", "bookkeep"]
    print(regime, "emissions", n, {k: round(int(buf[i]) / max(n, 1), 1) for i, k in enumerate(names)})
