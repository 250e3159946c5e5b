import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import gen_inputs as gi  # noqa: E402

import paper_2508_07014_b200 as pb  # noqa: E402
from paper_2508_07014_b200 import _lib  # noqa: E402
from paper_2508_07014_b200.table import _host_out  # noqa: E402

phrases, V = gi.corpus("p20k_v1024")
ctx = pb.ContextList([pb.Phrase(" ".join(map(str, p)), p) for p in phrases], min_chars=0)
tab = pb.compile_arc_table(pb.compute_fail_links(pb.build_prefix_tree(ctx, pb.TreeParams(), V)))
B = 8192
st = np.random.default_rng(0).integers(0, tab.num_states, size=B).astype(np.int32)
h = tab.device_table().handle


def t(fn, n=10):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


print("host_out alloc ms", t(lambda: _host_out(B, V)))
ps, pn = _host_out(B, V)
print("advance_host pinned ms", t(lambda: _lib.LIB.pgpb_advance_host(h, _lib.ptr(st), B, _lib.ptr(ps), _lib.ptr(pn), _lib.stream_ptr())))
qs, qn = np.empty((B, V), np.float32), np.empty((B, V), np.int32)
print("advance_host pageable ms", t(lambda: _lib.LIB.pgpb_advance_host(h, _lib.ptr(st), B, _lib.ptr(qs), _lib.ptr(qn), _lib.stream_ptr())))
print("get_scores_batch ms", t(lambda: pb.get_scores_batch(tab, st)))
d = torch.empty(B * V * 2, dtype=torch.float32, device="cuda")
hp = torch.empty(B * V * 2, dtype=torch.float32, pin_memory=True)
print("raw D2H 64MiB pinned ms", t(lambda: hp.copy_(d)))
print("range check ms", t(lambda: (st.min() < 0 or st.max() >= tab.num_states)))
