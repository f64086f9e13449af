#!/usr/bin/env python
"""Render `--warmup` + `--frames` frames of a config for ncu captures.

    ncu --set full -k regex:k_ -s <warmup*kernels_per_frame> python tools/profile_frame.py
(--api draw, the default, is the bench's piko_draw: k_setup<FUSED>, k_cm_scan,
k_cm_scatter, k_tile per frame on c3; --api indexed adds k_vertex)
Prints kernels_per_frame on stderr so the skip count can be derived.
"""
from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--bin", type=int, default=16)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--frames", type=int, default=1)
    ap.add_argument("--api", choices=["draw", "indexed"], default="draw",
                    help="piko_draw (the bench headline: fused vertex stage) or piko_draw_indexed")
    a = ap.parse_args()
    import torch

    import paper_1404_6293_b200 as piko
    import scenes
    s = scenes.make(a.config)
    v = torch.from_numpy(s.verts).cuda()
    i = torch.from_numpy(s.idx).cuda()
    r = piko.Renderer(s.W, s.H, a.bin)
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    for k in range(a.warmup + a.frames):
        flush.fill_(float(k))
        r.draw(v, i, s.mvp, s.light, indexed=a.api == "indexed")
    torch.cuda.synchronize()
    st = r.stats()
    print(f"stats {st}", file=sys.stderr)
    r.close()


if __name__ == "__main__":
    main()
