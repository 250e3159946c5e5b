"""Device-timed greedy CTC regimes (fused vs two-phase kernels), 20K tree, V=1024.

python scripts/ctc_regimes.py [B] [T]
"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen_inputs as gi  # noqa: E402
import paper_2508_07014_b200 as pb  # noqa: E402
from paper_2508_07014_b200.acoustic import synth_ctc_emissions  # noqa: E402
from paper_2508_07014_b200.context import Vocabulary  # noqa: E402


def table():
    phrases, V = gi.corpus(os.environ.get("PGPB_BENCH_CORPUS", "p20k_v1024"))
    ctx = pb.ContextList([pb.Phrase(" ".join(map(str, p)), p) for p in phrases], min_chars=0)
    return pb.compile_arc_table(pb.compute_fail_links(pb.build_prefix_tree(ctx, pb.TreeParams(), V))), V


def regimes(B, T, V, dev):
    g = torch.Generator(device=dev)
    g.manual_seed(1234)
    out = {}
    logits = torch.randn((B, T, V), generator=g, device=dev) * 2.0
    out["dense"] = torch.log_softmax(logits, -1).contiguous()
    logits[:, torch.arange(T, device=dev) % 4 != 0, 0] += 10.0
    out["blank3"] = torch.log_softmax(logits, -1).contiguous()
    del logits
    rng = np.random.default_rng(5)
    vocab = Vocabulary(tokens=tuple(str(i) for i in range(V)), blank_id=0)
    ems = []
    for _ in range(B):
        tgt = [int(x) for x in rng.integers(1, V, size=T // 4 + 1)]
        ems.append(synth_ctc_emissions(tgt, vocab, margin=0.5, seed=int(rng.integers(2**31)), boost_positions=[],
                                       blanks_between=3).logprobs[:T])
    out["clean"] = torch.from_numpy(np.stack(ems)).to(dev)
    return out


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for _ in range(reps):
            fn()
    gr.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    gr.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 200
    dev = torch.device("cuda")
    tab, V = table()
    only = os.environ.get("PGPB_REGIMES")
    impls = os.environ.get("PGPB_IMPLS", "fused,twophase").split(",")
    for name, lp in regimes(B, T, V, dev).items():
        if only and name not in only.split(","):
            continue
        row = {}
        for impl in impls:
            if impl == "twophase":
                os.environ["PGPB_CTC_TWOPHASE"] = "1"
            else:
                os.environ.pop("PGPB_CTC_TWOPHASE", None)
            for lam in (0.0, 1.0):
                cfg = pb.DecodeConfig(lam=lam)
                o = pb.ctc_greedy_device(lp, None, tab, cfg, 0)
                row[f"{impl}_lam{lam:g}_us"] = round(timeit(lambda: pb.ctc_greedy_device(lp, None, tab, cfg, 0, out=o)), 2)
        os.environ.pop("PGPB_CTC_TWOPHASE", None)
        row["fused_overhead"] = round(row["fused_lam1_us"] / row["fused_lam0_us"] - 1, 3)
        hbm = B * T * V * 4 / (row["fused_lam0_us"] * 1e-6) / 1e9
        row["fused_unboosted_GBps"] = round(hbm, 1)
        print(name, row, flush=True)


if __name__ == "__main__":
    main()
