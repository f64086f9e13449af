#!/usr/bin/env python
"""Small frames of every pipeline for compute-sanitizer runs:
    compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize.py
Renders c1 (64x64, 8x8 bins) and a 200x120 soup with the binned (count-matrix
and radix AssignBin), FreePipe and Baseline pipelines (two frames each,
forward shader cost on the second), the binned path with split bins (a dense
stack), a small Reyes patch scene (device Split/Dice), and checks each frame
against the CPU oracle."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1404_6293_b200 as piko  # noqa: E402
import scenes  # noqa: E402

oracle.build()
cases = [(scenes.scene_c1(), 8),
         (scenes.scene_soup(3000, 200, 120, seed=41, name="soup", bin_sizes=(16,)), 16),
         (scenes.scene_soup(6000, 64, 64, seed=43, name="dense", bin_sizes=(8,)), 8)]
for s, bw in cases:
    ref = oracle.render(s.verts, s.idx, s.mvp, s.light, s.W, s.H)
    v = torch.from_numpy(s.verts).cuda()
    i = torch.from_numpy(s.idx).cuda()
    for pipe in (piko.PIKO_PIPE_BINNED, "radix", piko.PIKO_PIPE_FREEPIPE, piko.PIKO_PIPE_BASELINE):
        os.environ["PIKO_CM"] = "0" if pipe == "radix" else "1"
        r = piko.Renderer(s.W, s.H, bw)
        os.environ.pop("PIKO_CM")
        if pipe != "radix":
            piko.piko_set_pipeline(r.ctx, pipe)
        for k in range(2):
            piko.piko_set_shader_cost(r.ctx, 8 * k, 1)
            r.draw(v, i, s.mvp, s.light)
        torch.cuda.synchronize()
        ok = (np.array_equal(r.primid().cpu().numpy(), ref["primid"])
              and np.array_equal(r.depth.cpu().numpy().view(np.uint32), ref["depth"].view(np.uint32)))
        print(f"{s.name} bin {bw} pipeline {pipe}: {'ok' if ok else 'MISMATCH'}", flush=True)
        assert ok
        r.close()
ps = scenes.scene_patches(n=2, seed=64, dice_px=4.0, W=128, H=96, name="patches")
G, pv, pi = oracle.dice(ps.patches, ps.mvp, ps.W, ps.H, ps.dice_px, ps.max_grid)
ref = oracle.render(pv, pi, ps.mvp, ps.light, ps.W, ps.H)
r = piko.Renderer(ps.W, ps.H, 32)
pt = torch.from_numpy(ps.patches).cuda()
for k in range(2):
    r.draw_patches(pt, ps.mvp, ps.light, ps.dice_px, ps.max_grid)
torch.cuda.synchronize()
ok = (np.array_equal(r.primid().cpu().numpy(), ref["primid"])
      and np.array_equal(r.depth.cpu().numpy().view(np.uint32), ref["depth"].view(np.uint32)))
print(f"reyes patches bin 32: {'ok' if ok else 'MISMATCH'}", flush=True)
assert ok
r.close()
print("sanitize frames done")
