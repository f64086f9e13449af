#!/usr/bin/env python
"""Frame-level DRAM traffic (BASELINE.md's measured-bytes definition) with ncu
range replay: every kernel of one steady-state frame inside one
cudaProfilerStart/Stop range, so one result covers the whole frame.  Three
ranges after the warm-up frames: (A) the frame alone, (B) an L2 flush alone,
(C) the frame followed by the flush; C - B adds the frame's dirty L2 lines
that are written back only after the frame.
    ncu --replay-mode range --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \\
        --csv --log-file out.csv python tools/frame_dram.py --config c3
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--bin", type=int, default=16)
    ap.add_argument("--indexed", action="store_true")
    a = ap.parse_args()
    import torch
    import paper_1404_6293_b200 as piko
    import scenes
    s = scenes.make(a.config)
    r = piko.Renderer(s.W, s.H, a.bin, sync="async")
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    if isinstance(s, scenes.PatchScene):
        pt = torch.from_numpy(s.patches).cuda()

        def frame():
            r.draw_patches(pt, s.mvp, s.light, s.dice_px, s.max_grid)
    else:
        v = torch.from_numpy(s.verts).cuda()
        i = torch.from_numpy(s.idx).cuda()

        def frame():
            r.draw(v, i, s.mvp, s.light, indexed=a.indexed)
    for k in range(5):
        flush.fill_(float(k))
        frame()
    piko.piko_finish(r.ctx)
    torch.cuda.synchronize()
    prof = torch.cuda.profiler
    flush.fill_(1.0)
    torch.cuda.synchronize()
    # (piko_finish outside the ranges: a range may not query events recorded
    # outside it, and the frame status ring is drained between them)
    prof.start(); frame(); torch.cuda.synchronize(); prof.stop()             # A
    assert piko.piko_finish(r.ctx) == piko.PIKO_OK
    prof.start(); flush.fill_(2.0); torch.cuda.synchronize(); prof.stop()    # B
    prof.start(); frame(); flush.fill_(3.0); torch.cuda.synchronize(); prof.stop()  # C
    assert piko.piko_finish(r.ctx) == piko.PIKO_OK
    print("ranges: A frame, B flush, C frame+flush", file=sys.stderr)


if __name__ == "__main__":
    main()
