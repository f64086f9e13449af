#!/usr/bin/env python
"""Pixel-shader complexity sweep (the paper's sec. 7.2.1 axis, P:1281-1294;
SURVEY 8(f) NEXT-3): ms/frame of the binned pipeline (LoadBalance: per-bin
CTAs), of FreePipe (DirectMap: the triangle's own thread) and of Baseline
(LoadBalance, one kernel per stage, fragments in HBM) as the per-fragment
shader cost grows, forward (every covered fragment pays, the paper's order:
shade before the depth test) and deferred (once per resolved pixel).
Protocol as tools/sweep.py (inputs in HBM, L2 flushed before each frame outside
its CUDA events, warm-up, median of 20).  Writes profiles/shader_sweep_<tag>.json."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1404_6293_b200 as piko  # noqa: E402
import scenes  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
cfgs = sys.argv[2].split(",") if len(sys.argv) > 2 else ["c2", "c3"]
iters_list = [0, 16, 64, 256, 1024]
steps, warm = 20, 3
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
res = []
for cfg in cfgs:
    s = scenes.make(cfg)
    v = torch.from_numpy(s.verts).cuda()
    i = torch.from_numpy(s.idx).cuda()
    for pipe in (piko.PIKO_PIPE_BINNED, piko.PIKO_PIPE_FREEPIPE, piko.PIKO_PIPE_BASELINE):
        r = piko.Renderer(s.W, s.H, 16)
        piko.piko_set_pipeline(r.ctx, pipe)
        for it in iters_list:
            for fwd in ((1, 0) if it else (0,)):
                piko.piko_set_shader_cost(r.ctx, it, fwd)
                piko.piko_set_sync(r.ctx, piko.PIKO_SYNC_CHECKED)
                for _ in range(warm):
                    r.draw(v, i, s.mvp, s.light)
                piko.piko_set_sync(r.ctx, piko.PIKO_SYNC_ASYNC)
                ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                      for _ in range(steps)]
                torch.cuda.synchronize()
                for k in range(steps):
                    flush.fill_(float(k))
                    ev[k][0].record()
                    r.draw(v, i, s.mvp, s.light)
                    ev[k][1].record()
                torch.cuda.synchronize()
                assert piko.piko_finish(r.ctx) == 0
                ms = sorted(a.elapsed_time(b) for a, b in ev)[steps // 2]
                res.append({"config": cfg, "pipeline": ("binned", "freepipe", "baseline")[pipe],
                            "shader_iters": it, "shading": "forward" if fwd else "deferred",
                            "median_ms": ms})
                print(res[-1], flush=True)
        r.close()
json.dump(res, open(os.path.join(ROOT, "profiles", f"shader_sweep_{tag}.json"), "w"), indent=1)
print("| config | shading | iters | binned ms | FreePipe ms | Baseline ms | FreePipe / binned | Baseline / binned |")
print("|---|---|---|---|---|---|---|---|")
for x in res:
    if x["pipeline"] != "binned":
        continue
    o = {y["pipeline"]: y["median_ms"] for y in res if y["config"] == x["config"]
         and y["shader_iters"] == x["shader_iters"] and y["shading"] == x["shading"]}
    print(f"| {x['config']} | {x['shading'] if x['shader_iters'] else '-'} | {x['shader_iters']} | "
          f"{x['median_ms']:.3f} | {o['freepipe']:.3f} | {o['baseline']:.3f} | "
          f"{o['freepipe'] / x['median_ms']:.2f} | {o['baseline'] / x['median_ms']:.2f} |")
