"""Small driver for ncu captures: advance (config 5) and greedy CTC launches."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import gen_inputs as gi  # noqa: E402

import paper_2508_07014_b200 as pb  # noqa: E402
from paper_2508_07014_b200 import _lib  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "advance"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
phrases, V = gi.corpus("p20k_v1024")
ctx = pb.ContextList([pb.Phrase(" ".join(map(str, p)), p) for p in phrases], min_chars=0)
tab = pb.compile_arc_table(pb.compute_fail_links(pb.build_prefix_tree(ctx, pb.TreeParams(), V)))
rng = np.random.default_rng(0)
if what in ("advance", "chain"):
    B = 8192
    st = [torch.from_numpy(rng.integers(0, tab.num_states, size=B).astype(np.int32)).cuda() for _ in range(4)]
    outs = [(torch.empty((B, V), device="cuda"), torch.empty((B, V), dtype=torch.int32, device="cuda")) for _ in range(4)]
    h = tab.device_table().handle
    fn = _lib.LIB.pgpb_advance if what == "advance" else _lib.LIB.pgpb_advance_chain
    for i in range(reps):
        s, n = outs[i % 4]
        _lib.check(fn(h, st[i % 4].data_ptr(), B, s.data_ptr(), n.data_ptr(), _lib.stream_ptr()))
elif what == "greedy":
    B, T = 128, 200
    lp = torch.log_softmax(torch.randn((B, T, V), device="cuda") * 2.0, dim=-1).contiguous()
    for i in range(reps):
        pb.ctc_greedy_device(lp, None, tab, pb.DecodeConfig(lam=1.0), 0)
torch.cuda.synchronize()
print("done", what)
