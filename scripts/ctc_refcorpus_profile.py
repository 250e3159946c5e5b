"""Greedy CTC on the reference's overhead corpus (25 x ~1800 frames):
device time of phase A / walker variants and the walker's checkpoint
timeline (needs PGPB_LIB_PATH=.../libpgpb_prof.so for the counters;
scripts/experiments/build_prof_lib.sh)."""
import ctypes
import os
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
from paper_2508_07014_b200.acoustic import synth_ctc_emissions  # noqa: E402
from paper_2508_07014_b200.context import Vocabulary  # noqa: E402

phrases, V = gi.corpus("p20k_v1024")
ctx = pb.ContextList([pb.Phrase(" ".join(map(str, p)), p) for p in phrases], min_chars=0)
tab = pb.compile_arc_table(pb.compute_fail_links(pb.build_prefix_tree(ctx, pb.TreeParams(), V)))
vocab = Vocabulary(tokens=tuple(str(i) for i in range(V)), blank_id=0)
if len(sys.argv) > 1 and sys.argv[1] == "clean200":  # the bench's clean regime shape
    rng = np.random.default_rng(4242)
    targets = [[int(x) for x in rng.integers(1, V, size=51)] for _ in range(128)]
    seeds = [int(rng.integers(2**31)) for _ in range(128)]
    ems = [synth_ctc_emissions(tg, vocab, margin=0.5, seed=sd, boost_positions=[], blanks_between=3).logprobs[:200]
           for tg, sd in zip(targets, seeds)]
else:
    targets, seeds, _ = gi.reference_overhead_corpus()
    ems = [synth_ctc_emissions(tg, vocab, margin=0.5, seed=sd, boost_positions=[], blanks_between=3).logprobs
           for tg, sd in zip(targets, seeds)]
lens = np.array([e.shape[0] for e in ems], np.int32)
pad = np.zeros((len(ems), int(lens.max()), V), np.float32)
for i, e in enumerate(ems):
    pad[i, :e.shape[0]] = e
lp = torch.from_numpy(pad).cuda()
ln = torch.from_numpy(lens).cuda()


def timed(cfg, reps=10):
    o = pb.ctc_greedy_device(lp, ln, tab, cfg, 0)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            pb.ctc_greedy_device(lp, ln, tab, cfg, 0, out=o)
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


for key, vals in [("", [0]), ("ctc.seq", [2]), ("ctc.consumers", [3, 5])]:
    for v in vals:
        if key:
            _lib.set_tuning(key, v)
        print(key or "auto", v, "unboosted us", round(timed(pb.DecodeConfig(lam=0.0)), 2), "boosted us",
              round(timed(pb.DecodeConfig(lam=1.0)), 2), flush=True)
        if key:
            _lib.set_tuning(key, 0)

if hasattr(_lib.LIB, "pgpb_debug_ctc_fused_profile"):
    f = _lib.LIB.pgpb_debug_ctc_fused_profile
    f.argtypes = [ctypes.c_void_p, ctypes.c_int]
    buf = np.zeros(256, np.uint64)
    cfg = pb.DecodeConfig(lam=1.0)
    pb.ctc_greedy_device(lp, ln, tab, cfg, 0)
    torch.cuda.synchronize()
    f(buf.ctypes.data, 1)
    pb.ctc_greedy_device(lp, ln, tab, cfg, 0)
    torch.cuda.synchronize()
    f(buf.ctypes.data, 1)
    names = ["fixup_rounds", "r0_steps", "fix_steps", "warp_dec", "rescans", "cyc_prod", "cyc_r0", "cyc_fix",
             "cyc_tail", "segments", "gathers", "lane_dec_n", "lane_dec_cyc", "am_sum_cyc", "warp_dec_n",
             "warp_dec_cyc"]
    print({k: int(buf[i]) for i, k in enumerate(names)})
    print("timeline (CTA 0, cycles since entry): prologue", int(buf[200]), "wait released", int(buf[201]),
          "staged", int(buf[202]), "mode", int(buf[203]), "guessed", int(buf[204]), "round0", int(buf[205]),
          "walk done", int(buf[206]), "sums", int(buf[207]), "end", int(buf[208]), "scanback", int(buf[212]),
          "rt1 issued", int(buf[213]), "rt1 used", int(buf[214]))
    print("round0 per warp: max", int(buf[194]), "mean", int(buf[195]) / max(1, int(buf[196])))
    names2 = {0: "none", 1: "fast", 3: "semi", 5: "root", 8: "scan", 9: "fast>scan", 11: "semi>scan"}
    print("lane paths (all CTAs):", {f"{names2.get(k, k)}:{'ok' if r else 'fail'}": int(buf[160 + 2 * k + r])
                                     for k in range(16) for r in (0, 1) if buf[160 + 2 * k + r]})
