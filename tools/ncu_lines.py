#!/usr/bin/env python
"""Warp-stall samples aggregated per CUDA source line (needs -lineinfo).
usage: python tools/ncu_lines.py report.ncu-rep kernel_regex [N] [function-substring] [--instr]
--instr ranks lines by warp instructions executed instead of stall samples."""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
want = sys.argv[4] if len(sys.argv) > 4 and not sys.argv[4].startswith("--") else None
col = "Instructions Executed" if "--instr" in sys.argv else "Warp Stall Sampling (All Samples)"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
sections, cur = [], None
for r in rows:
    if r and r[0] == "Function Name":
        cur = {"name": r[1], "rows": []}
        sections.append(cur)
    elif cur is not None:
        cur["rows"].append(r)
for sec in sections:
    if want and want not in sec["name"]:
        continue
    rs = sec["rows"]
    hdr_i = next(i for i, r in enumerate(rs) if r and r[0] == "Line No")
    h = rs[hdr_i]
    ismp = h.index(col)
    lines = {}
    for r in rs[hdr_i + 1:]:
        if len(r) > ismp and r[0]:
            try:
                lines[(int(r[0]), r[1].strip())] = int(r[ismp] or 0)
            except ValueError:
                pass
    tot = sum(lines.values()) or 1
    print(f"## {sec['name']}  total {col}: {tot}")
    for (ln, src), v in sorted(lines.items(), key=lambda kv: -kv[1])[:n]:
        print(f"{v:6d} {100*v/tot:5.1f}%  L{ln:<5d} {src[:100]}")
    if want:
        break
