"""Bench-shape workloads for one-kernel ncu captures (scripts/gpu_ncu_kernels.sh).

python scripts/ncu_workloads.py {config3|config3_unfused|config4|aed_greedy|beam_api|hits|label_loop|greedy_host|
                                 advance_single|table_helpers|ctc_clean_boosted|ctc_clean_unboosted}
"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import bench_workloads as bw  # noqa: E402
import gen_inputs as gi  # noqa: E402

import paper_2508_07014_b200 as pb  # noqa: E402

dev = torch.device("cuda", 0)
what = sys.argv[1]
if what == "config3":
    from paper_2508_07014_b200.beams import TransducerBeamDecoder

    model, tab, enc = bw.config3(dev)
    c = bw.C3
    dec = TransducerBeamDecoder(model, tab, pb.DecodeConfig(lam=1.0, beam_size=4, max_symbols_per_frame=5), c["B"],
                                c["T"], use_graph=False)
    dec.run(enc, torch.full((c["B"],), 20))
elif what in ("config4", "aed_greedy"):
    from paper_2508_07014_b200.beams import AEDBeamDecoder, AEDGreedyDecoder

    model, tab, mem = bw.config4(dev)
    c = bw.C4
    V = tab.vocab_size
    if what == "config4":
        AEDBeamDecoder(model, tab, pb.DecodeConfig(lam=1.0, beam_size=4), c["B"], max_len=c["max_len"], eos=V - 1,
                       use_graph=False).run(mem)
    else:
        AEDGreedyDecoder(model, tab, pb.DecodeConfig(lam=1.0, beam_size=1), c["B"], max_len=c["max_len"], eos=V - 1,
                         use_graph=False).run(mem)
elif what == "beam_api":
    tab, V = bw.table("p5k_v1024")
    rng = np.random.default_rng(77)
    em = pb.EmissionMatrix(gi.random_emissions(rng, 20, V), blank_id=0)
    pb.ctc_beam_boosted(em, tab, pb.DecodeConfig(lam=1.0, beam_size=4))
elif what == "hits":
    from paper_2508_07014_b200.evaluation import keyphrase_hits_device

    rng = np.random.default_rng(3)
    vocab = [f"w{i}" for i in range(500)]
    U = 20000
    refs = [[vocab[int(j)] for j in rng.integers(0, 500, size=int(rng.integers(5, 40)))] for _ in range(U)]
    hyps = [[vocab[int(j)] for j in rng.integers(0, 500, size=int(rng.integers(5, 40)))] for _ in range(U)]
    phrases = [" ".join(vocab[int(j)] for j in rng.integers(0, 500, size=int(rng.integers(1, 4)))) for _ in range(2000)]
    keyphrase_hits_device(refs, hyps, phrases)
elif what == "label_loop":
    from paper_2508_07014_b200.rnnt import LabelLoopingDecoder

    model, tab, enc_proj = bw.config2(dev)
    c = bw.C2
    LabelLoopingDecoder(model, tab, pb.DecodeConfig(lam=1.0), c["B"], c["T"], use_graph=False).decode(enc_proj)
elif what == "greedy_host":  # transducer_greedy_boosted with a host StepModel (pgpb_greedy_step)
    tab, V = bw.table("p5k_v1024")
    rng = np.random.default_rng(5)
    rows, default = gi.random_transducer_rows(rng, V)
    m = pb.TableStepModel(flavor="transducer", default_row=default, rows=rows)
    pb.transducer_greedy_boosted(m, 30, 0, tab, pb.DecodeConfig(lam=1.0))
elif what == "advance_single":  # get_scores_batch on device tensors, 8192 rows (advance_v6_kernel)
    tab, V = bw.table("p20k_v1024")
    st = torch.from_numpy(np.random.default_rng(1).integers(0, tab.num_states, size=8192).astype(np.int32)).to(dev)
    for _ in range(4):
        pb.get_scores_batch(tab, st)
elif what == "table_helpers":  # per-table precomputations (row_max, final_bonus, backoff_total)
    tab, V = bw.table("p20k_v1024")
    dt = tab.device_table(0)
    dt.row_max(), dt.final_bonus(), dt.backoff_total()
elif what == "config3_unfused":  # beam_hidden_kernel + log_softmax_bf16_kernel (the unfused wave)
    from paper_2508_07014_b200.beams import TransducerBeamDecoder

    model, tab, enc = bw.config3(dev)
    c = bw.C3
    dec = TransducerBeamDecoder(model, tab, pb.DecodeConfig(lam=1.0, beam_size=4, max_symbols_per_frame=5), c["B"],
                                c["T"], use_graph=False, fused=False)
    dec.run(enc, torch.full((c["B"],), 4))
torch.cuda.synchronize()
print("ok", what)
if what.startswith("ctc_clean"):
    sys.path.insert(0, str(ROOT / "scripts"))
    import ctc_regimes as cr

    tab, V = cr.table()
    lp = cr.regimes(128, 200, V, dev)["clean"]
    lam = 0.0 if what.endswith("unboosted") else 1.0
    for _ in range(3):
        pb.ctc_greedy_device(lp, None, tab, pb.DecodeConfig(lam=lam), 0)
    torch.cuda.synchronize()
    print("ok", what)
