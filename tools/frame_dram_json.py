#!/usr/bin/env python
"""profiles/traffic_frame_<cfg>_b<bin>.json from the ncu range-replay CSV of
tools/frame_dram.py (ranges: A frame, B flush, C frame + flush).
usage: python tools/frame_dram_json.py frame_dram.csv cfg bin"""
import csv
import json
import os
import sys

path, cfg, bw = sys.argv[1], sys.argv[2], sys.argv[3]
vals = {}
for r in csv.reader(open(path)):
    if len(r) > 12 and r[0].isdigit():
        vals.setdefault(int(r[0]), {})[r[10]] = float(r[12])
rng = [vals[k] for k in sorted(vals)]
def tot(d):
    return d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
out = {"frame_A_bytes": int(tot(rng[0])), "frame_A_read": int(rng[0]["dram__bytes_read.sum"]),
       "frame_A_write": int(rng[0]["dram__bytes_write.sum"])}
if len(rng) >= 3:
    out["flush_B_bytes"] = int(tot(rng[1]))
    out["frame_plus_flush_C_bytes"] = int(tot(rng[2]))
    out["frame_with_writebacks_bytes"] = int(tot(rng[2]) - tot(rng[1]))
out["frame_bytes"] = max(out["frame_A_bytes"], out.get("frame_with_writebacks_bytes", 0))
out["_note"] = ("ncu --replay-mode range over one steady-state frame (all its kernels in one range): "
                "A = the frame alone; C - B = frame + flush minus flush alone, i.e. including the "
                "frame's dirty L2 lines written back later. frame_bytes = max(A, C - B).")
out["_source"] = os.path.basename(path)
dst = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                   f"traffic_frame_{cfg}_b{bw}.json")
json.dump(out, open(dst, "w"), indent=1)
print(json.dumps(out))
