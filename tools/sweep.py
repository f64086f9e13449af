#!/usr/bin/env python
"""Design sweep (BASELINE.json configs[2] bin-size sweep):
ms/frame of the binned pipeline at bins 8/16/32/64 and of the FreePipe
alternative on c2, c3, c4, with bench.py's protocol (inputs in
HBM, L2 flushed before each frame outside its CUDA events, warm-up).
Writes profiles/sweep_<tag>.json and prints a markdown table."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1404_6293_b200 as piko  # noqa: E402
import scenes  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
steps, warm = 20, 4
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
res = []
for cfg in ("c2", "c3", "c4"):
    s = scenes.make(cfg)
    v = torch.from_numpy(s.verts).cuda()
    i = torch.from_numpy(s.idx).cuda()
    for pipe, bw in [(0, 8), (0, 16), (0, 32), (0, 64), (1, 16)]:
        r = piko.Renderer(s.W, s.H, bw)
        piko.piko_set_pipeline(r.ctx, pipe)
        for _ in range(warm):
            r.draw(v, i, s.mvp, s.light)
        piko.piko_set_sync(r.ctx, piko.PIKO_SYNC_ASYNC)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        torch.cuda.synchronize()
        for k in range(steps):
            flush.fill_(float(k))
            ev[k][0].record()
            r.draw(v, i, s.mvp, s.light)
            ev[k][1].record()
        torch.cuda.synchronize()
        assert piko.piko_finish(r.ctx) == 0
        ms = sorted(a.elapsed_time(b) for a, b in ev)[steps // 2]
        st = r.stats()
        res.append({"config": cfg, "pipeline": "freepipe" if pipe else "binned", "bin": bw if not pipe else None,
                    "n_tris": s.n_tris, "n_pairs": st["n_pairs"] if not pipe else None,
                    "median_ms": ms, "mtri_s": s.n_tris / ms / 1e3})
        r.close()
        print(res[-1], flush=True)
json.dump(res, open(os.path.join(ROOT, "profiles", f"sweep_{tag}.json"), "w"), indent=1)
print("| config | pipeline | bin | pairs | median ms/frame | Mtri/s |")
print("|---|---|---|---|---|---|")
for x in res:
    print(f"| {x['config']} | {x['pipeline']} | {x['bin'] or '-'} | {x['n_pairs'] or '-'} | "
          f"{x['median_ms']:.3f} | {x['mtri_s']:.0f} |")
