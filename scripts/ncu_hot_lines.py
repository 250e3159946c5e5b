"""Per-CUDA-line warp-stall samples of an ncu report (top N lines).
python scripts/ncu_hot_lines.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, agg, tot = None, {}, 0
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    i = hdr.index("Warp Stall Sampling (All Samples)")
    try:
        v = int(r[i])
    except ValueError:
        continue
    key = (fname, int(r[0]))
    agg.setdefault(key, [0, r[1].strip()[:90]])
    agg[key][0] += v
    tot += v
print(f"total samples {tot}")
for (f, ln), (v, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:N]:
    print(f"{v:6d} {100.0 * v / max(tot, 1):5.1f}%  {f}:{ln}  {src}")
