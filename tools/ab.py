#!/usr/bin/env python
"""A/B timing of compile-time variants of libpiko (experiments only).
usage: python tools/ab.py CONFIG BIN 'name=-DFLAG ...' ['name2:alt/kernels.cu=...' ...]
Each variant is compiled to /tmp and timed in its own process: median frame
time over 30 frames (L2 flushed before each, CUDA events on the draw stream)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def build(name, flags, alt=None):
    import __graft_entry__ as ge
    lib = f"/tmp/libpiko_ab_{name}.so"
    objs = []
    for src in sorted({src for src, _, _ in ge.SOURCES}):  # one TU per source (no tile split)
        o = f"/tmp/{src}.ab_{name}.o"
        path = alt if (alt and src == "kernels.cu") else os.path.join(ge.CSRC, src)
        subprocess.check_call([ge._nvcc(), *ge.NVCC_FLAGS, *flags, "-I", ge.CSRC, "-c", path, "-o", o])
        objs.append(o)
    subprocess.check_call([ge._nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs,
                           "-o", lib, "-ldl", "-lcudart"])
    return lib


def run(lib, cfg, bw):
    import numpy as np
    import torch
    import paper_1404_6293_b200 as piko
    piko.LIB_PATH = lib
    piko._lib = piko.lib = piko._load()
    import scenes
    s = scenes.make(cfg)
    v = torch.from_numpy(s.verts).cuda()
    i = torch.from_numpy(s.idx).cuda()
    r = piko.Renderer(s.W, s.H, bw)
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream()
    ts = []
    for k in range(40):
        flush.fill_(float(k))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        r.draw(v, i, s.mvp, s.light)
        e1.record(st)
        torch.cuda.synchronize()
        if k >= 10:
            ts.append(e0.elapsed_time(e1) * 1000.0)
    ts = np.array(ts)
    print(f"median {np.median(ts):.1f} us  p10 {np.percentile(ts, 10):.1f}  p90 {np.percentile(ts, 90):.1f}")


if __name__ == "__main__":
    if sys.argv[1] == "--run":
        run(sys.argv[2], sys.argv[3], int(sys.argv[4]))
        sys.exit(0)
    cfg, bw = sys.argv[1], int(sys.argv[2])
    libs = []
    for spec in sys.argv[3:]:
        name, _, fl = spec.partition("=")
        name, _, alt = name.partition(":")  # name:ALT_KERNELS_CU (another kernels.cu)
        libs.append((name, build(name, [f for f in fl.split() if f], alt or None)))
    for rep in range(2):
        for name, lib in libs:
            out = subprocess.run([sys.executable, __file__, "--run", lib, cfg, str(bw)], capture_output=True, text=True)
            print(f"{cfg} b{bw} {name:12s} {out.stdout.strip()} {out.stderr.strip()[-300:] if out.returncode else ''}", flush=True)
