"""Write profiles/advance_ncu_summary.json (bench.py's roofline.traffic) from
a `--set full` capture of the headline kernel: DRAM read + write bytes of
the launch."""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
hdr, units, vals = r[0], r[1], r[2]
idx = {h: i for i, h in enumerate(hdr)}
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3}


def get(m):
    return float(vals[idx[m]].replace(",", "")) * UNIT.get(units[idx[m]], 1.0)


rd, wr, dur = get("dram__bytes_read.sum"), get("dram__bytes_write.sum"), get("gpu__time_duration.sum")
d = {"kernel": vals[idx["Kernel Name"]].split("(")[0],
     "capture": f"ncu --set full --clock-control none, one launch of the bench command ({rep.split('/')[-1]})",
     "dram_bytes_per_launch": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr, "duration_us": dur,
     "grid": vals[idx["launch__grid_size"]], "registers": vals[idx["launch__registers_per_thread"]],
     "note": "DRAM traffic within the launch (ncu replays are serialised and cold); output lines still dirty in "
             "L2 at the end of the launch are written back during the next one"}
json.dump(d, open("profiles/advance_ncu_summary.json", "w"), indent=1)
print(json.dumps(d, indent=1))
