"""Fused CTC config sweep (env knobs), device-timed, 20K tree, B=128 x T=200."""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CODE = r'''
import sys, os
sys.path.insert(0, "scripts")
import ctc_regimes as cr, torch, paper_2508_07014_b200 as pb
tab, V = cr.table()
regs = cr.regimes(128, 200, V, torch.device("cuda"))
out = []
for name in ("clean", "dense"):
    lp = regs[name]
    for lam in (0.0, 1.0):
        cfg = pb.DecodeConfig(lam=lam)
        o = pb.ctc_greedy_device(lp, None, tab, cfg, 0)
        out.append("%s/%g=%.1f" % (name, lam, cr.timeit(lambda: pb.ctc_greedy_device(lp, None, tab, cfg, 0, out=o))))
print(os.environ.get("TAG"), " ".join(out), flush=True)
'''
for env in sys.argv[1:]:
    e = dict(os.environ)
    kv = dict(x.split("=") for x in env.split(",") if x)
    e.update(kv)
    e["TAG"] = env
    subprocess.run([sys.executable, "-c", CODE], env=e, cwd=ROOT)
