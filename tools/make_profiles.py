#!/usr/bin/env python
"""Summarise ncu captures into profiles/ (tracked): per-kernel launch shares from
a gpu__time_duration launch list, and per-kernel DRAM traffic / utilisation from
a --set full report.  Also writes profiles/traffic_<cfg>_b<bin>.json (DRAM bytes
per launch by bench stage) which bench.py reports as roofline.traffic.
usage: python tools/make_profiles.py <tag> <launches.csv> <full.ncu-rep> <cfg> <bin>"""
import csv
import io
import json
import os
import subprocess
import sys

tag, launches, rep, cfg, bw = sys.argv[1:6]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out_dir = os.path.join(ROOT, "profiles")
os.makedirs(out_dir, exist_ok=True)

def kname(full):
    """'void piko::k_radix_pass<(bool)1>(piko::RadixArgs)' -> 'piko::k_radix_pass<(bool)1>'"""
    full = full.replace("void ", "")
    return full[:full.rfind("(")] if full.endswith(")") else full


def stage(name):
    base = name.split("<")[0].split("::")[-1]
    if base == "k_radix_pass":  # template argument EXPAND: pass 0 vs passes >= 1
        return "expand" if any(t in name for t in ("<(bool)1>", "<true>", "<1>")) else "sort"
    return {"k_vertex": "vertex", "k_setup": "setup", "k_tile": "tile", "k_resolve": "resolve",
            "k_bin_scan": "expand", "k_index_max": "vertex", "k_cm_scan": "expand",
            "k_cm_scatter": "sort", "k_shade": "resolve", "k_dice_rate": "dice",
            "k_dice": "dice"}.get(base)


rows = [r for r in csv.reader(open(launches)) if r and not r[0].startswith("==")]
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
tot = {}
for r in rows[1:]:
    if stage(kname(r[ki])) is not None:
        name = kname(r[ki])
        tot.setdefault(name, []).append(float(r[vi]) / 1000.0)
lines = [f"# ncu launch list ({tag}): gpu__time_duration per launch, cold-cache, serialised",
         "# kernel, launches, mean_us, share_of_frame"]
frame = sum(sum(v) / len(v) for v in tot.values())
for k, v in sorted(tot.items(), key=lambda kv: -sum(kv[1]) / len(kv[1])):
    m = sum(v) / len(v)
    lines.append(f"{k}, {len(v)}, {m:.2f}, {m / frame:.3f}")
open(os.path.join(out_dir, f"launches_{tag}.txt"), "w").write("\n".join(lines) + "\n")

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
     "sm__throughput.avg.pct_of_peak_sustained_elapsed",
     "smsp__issue_active.avg.pct_of_peak_sustained_active",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
     "launch__grid_size"]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(M)],
                     capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
hh, units = rr[0], rr[1]
cols = [hh.index(m) for m in M if m in hh]
k2 = hh.index("Kernel Name")
summ = [f"# ncu --set full ({tag}), one launch per kernel of one frame ({cfg}, {bw}x{bw} bins)",
        "# kernel, " + ", ".join(f"{hh[c]} [{units[c]}]" for c in cols)]
traffic = {}
for r in rr[2:]:
    name = kname(r[k2])
    summ.append(name + ", " + ", ".join(r[c] for c in cols))
    st = stage(name)
    if st:
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = float(r[cols[1]]) * mult.get(units[cols[1]], 1)
        wr = float(r[cols[2]]) * mult.get(units[cols[2]], 1)
        traffic[st] = traffic.get(st, 0) + rd + wr
open(os.path.join(out_dir, f"ncu_full_{tag}.txt"), "w").write("\n".join(summ) + "\n")
json.dump({**{k: int(v) for k, v in traffic.items()}, "_source": f"profiles/ncu_full_{tag}.txt",
           "_note": "dram__bytes_read.sum + dram__bytes_write.sum per launch, ncu --set full "
                    "(cold caches: every kernel starts with an empty L2)"},
          open(os.path.join(out_dir, f"traffic_{cfg}_b{bw}.json"), "w"), indent=1)
print("\n".join(lines))
print("\n".join(summ))
