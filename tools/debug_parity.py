#!/usr/bin/env python
"""Render a config on the GPU and report where it differs from the oracle."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import paper_1404_6293_b200 as piko
import scenes

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--bin", type=int, default=32)
ap.add_argument("--repeat", type=int, default=3)
a = ap.parse_args()
s = scenes.make(a.config)
ref = oracle.render(s.verts, s.idx, s.mvp, s.light, s.W, s.H, want_covcount=True)
ostart, oprims = oracle.bins(s.verts, s.idx, s.mvp, s.W, s.H, a.bin, a.bin)
v = torch.from_numpy(s.verts).cuda()
i = torch.from_numpy(s.idx).cuda()
r = piko.Renderer(s.W, s.H, a.bin)
piko.piko_set_debug(r.ctx, 1)
for rep in range(a.repeat):
    r.draw(v, i, s.mvp, s.light)
    torch.cuda.synchronize()
    prim = r.primid().cpu().numpy()
    cov = r.coverage().cpu().numpy().view(np.uint32)
    st, pr = r.bins()
    st, pr = st.cpu().numpy(), pr.cpu().numpy()
    bad = np.argwhere(prim != ref["primid"])
    badc = np.argwhere(cov != ref["covcount"])
    print(f"rep {rep}: primid mismatches {len(bad)}, coverage mismatches {len(badc)}, "
          f"bins equal {np.array_equal(st, ostart) and np.array_equal(pr, oprims)}")
    for y, x in bad[:8]:
        b = (y // a.bin) * (-(-s.W // a.bin)) + x // a.bin
        print(f"  px ({x},{y}) bin {b}: gpu {prim[y, x]} oracle {ref['primid'][y, x]} "
              f"cov gpu {cov[y, x]} oracle {ref['covcount'][y, x]}")
    if not np.array_equal(st, ostart):
        d = np.argwhere(st != ostart)[:5].ravel()
        print("  bin_start differs at", d, st[d], ostart[d])
    elif not np.array_equal(pr, oprims):
        d = np.argwhere(pr != oprims)[:5].ravel()
        print("  bin_prims differs at", d, pr[d], oprims[d])
