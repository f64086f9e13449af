#!/usr/bin/env python
"""Top SASS instructions by warp-stall samples from an ncu report.
usage: python tools/ncu_hot.py report.ncu-rep kernel_regex [N]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ia, isrc, ismp = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
iex = h.index("Instructions Executed")
data = []
for r in rows[2:]:
    if len(r) <= max(ismp, iex):
        continue
    try:
        data.append((int(r[ismp] or 0), r[ia], r[isrc], r[iex]))
    except ValueError:
        pass
tot = sum(d[0] for d in data) or 1
print(f"total samples {tot}")
for d in sorted(data, reverse=True)[:n]:
    print(f"{d[0]:6d} {100*d[0]/tot:5.1f}%  {d[1]}  exec={d[3]:>8}  {d[2][:90]}")
