#!/usr/bin/env python
"""Warp-stall samples aggregated per CUDA source line (needs -lineinfo).
usage: python tools/ncu_lines.py report.ncu-rep kernel_regex [N]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hdr_i]
ismp = h.index("Warp Stall Sampling (All Samples)")
lines, cur = {}, None
for r in rows[hdr_i + 1:]:
    if len(r) <= ismp:
        continue
    if r[0]:                      # a source line row (aggregate of its SASS)
        try:
            lines[(int(r[0]), r[1].strip())] = int(r[ismp] or 0)
        except ValueError:
            pass
tot = sum(lines.values()) or 1
print(f"total samples {tot}")
for (ln, src), v in sorted(lines.items(), key=lambda kv: -kv[1])[:n]:
    print(f"{v:6d} {100*v/tot:5.1f}%  L{ln:<5d} {src[:100]}")
