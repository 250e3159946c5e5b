"""Summarise ncu reports (duration, DRAM bytes, bandwidth, L2 hit rate,
occupancy, registers) into a markdown table: python scripts/ncu_summary.py a.ncu-rep ..."""
import csv
import io
import subprocess
import sys

M = {
    "dur_us": ("gpu__time_duration.sum", 1e-3),
    "dram_rd_MB": ("dram__bytes_read.sum", 1e-6),
    "dram_wr_MB": ("dram__bytes_write.sum", 1e-6),
    "dram_GBps": ("dram__bytes.sum.per_second", 1e-9),
    "l2_hit_%": ("lts__t_sector_hit_rate.pct", 1.0),
    "sm_thru_%": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "mem_thru_%": ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "occ_%": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "regs": ("launch__registers_per_thread", 1.0),
    "grid": ("launch__grid_size", 1.0),
    "block": ("launch__block_size", 1.0),
}
UNIT = {"ns": 1.0, "us": 1e3, "ms": 1e6, "usecond": 1e3, "nsecond": 1.0, "msecond": 1e6,
        "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
        "byte/second": 1.0, "Kbyte/second": 1e3, "Mbyte/second": 1e6, "Gbyte/second": 1e9, "Tbyte/second": 1e12,
        "B/s": 1.0, "KB/s": 1e3, "MB/s": 1e6, "GB/s": 1e9, "TB/s": 1e12}

rows = []
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    if len(r) < 3:
        continue
    hdr, units, vals = r[0], r[1], r[2]
    idx = {h: i for i, h in enumerate(hdr)}
    name = vals[idx.get("Kernel Name", 0)][:60]
    d = {"report": rep.split("/")[-1], "kernel": name}
    for k, (metric, scale) in M.items():
        if metric in idx:
            v = vals[idx[metric]].replace(",", "")
            try:
                x = float(v) * UNIT.get(units[idx[metric]], 1.0)
                if k == "dur_us":
                    x = x / 1e3
                elif k.endswith("_MB"):
                    x = x / 1e6
                elif k == "dram_GBps":
                    x = x / 1e9
                d[k] = round(x, 2)
            except ValueError:
                d[k] = v
    if isinstance(d.get("dur_us"), float) and isinstance(d.get("dram_rd_MB"), float):
        d["dram_GBps"] = round((d["dram_rd_MB"] + d.get("dram_wr_MB", 0.0)) / d["dur_us"] * 1e3, 1)
    rows.append(d)
keys = ["report", "kernel"] + list(M)
print("| " + " | ".join(keys) + " |")
print("|" + "---|" * len(keys))
for d in rows:
    print("| " + " | ".join(str(d.get(k, "")) for k in keys) + " |")
