import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, torch
import bench, bench_workloads as bw
tab, V = bw.table("p20k_v1024")
for regime, lp, lens in bench._ctc_regimes(128, 200, V, torch.device("cuda", 0), 0):
    if regime.startswith("ref_corpus"):
        ln = lens.cpu().numpy(); host = lp.cpu().numpy()
        for _ in range(2):
            print(bench.ctc_reference_protocol([x[:n] for x, n in zip(host, ln)], tab), flush=True)
