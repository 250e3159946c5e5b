"""Per-SASS-instruction warp-stall samples of an ncu report, grouped by CUDA
line ranges: python scripts/ncu_sass_hot.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
iS, iE = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
stall = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[iS]) for r in data)
agg = {h: sum(int(r[hdr.index(h)]) for r in data) for h in stall}
print("samples", tot, "instructions executed", sum(int(r[iE]) for r in data))
print("by reason", sorted(((v, k[6:]) for k, v in agg.items()), reverse=True)[:8])
for r in sorted(data, key=lambda r: -int(r[iS]))[:N]:
    rs = sorted(((int(r[hdr.index(h)]), h[6:]) for h in stall), reverse=True)[:2]
    print(r[0][-5:], r[iS], r[iE], r[1].strip()[:70], rs)
