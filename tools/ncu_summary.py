#!/usr/bin/env python
"""One line per kernel launch from an ncu report: time, DRAM bytes, SM/issue %, regs, grid.
usage: python tools/ncu_summary.py report.ncu-rep [--csv out.csv]"""
import csv
import io
import subprocess
import sys

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "sm__throughput.avg.pct_of_peak_sustained_elapsed",
     "smsp__issue_active.avg.pct_of_peak_sustained_active",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
     "launch__grid_size", "lts__t_bytes.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(M)],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
ki = h.index("Kernel Name")
cols = [h.index(m) for m in M if m in h]
lines = []
hdr = ["kernel"] + [f"{h[c]} [{units[c]}]" for c in cols]
for r in rows[2:]:
    lines.append([r[ki].split("(")[0][:40]] + [r[c] for c in cols])
w = csv.writer(sys.stdout)
w.writerow(hdr)
for l in lines:
    w.writerow(l)
if "--csv" in sys.argv:
    with open(sys.argv[sys.argv.index("--csv") + 1], "w") as f:
        cw = csv.writer(f)
        cw.writerow(hdr)
        cw.writerows(lines)
