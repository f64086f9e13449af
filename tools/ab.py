#!/usr/bin/env python
"""A/B timing of compile-time variants of libpiko (experiments only).
usage: python tools/ab.py CONFIG BIN 'name=-DFLAG ...' ['name2:alt/kernels.cu=...' ...]
       python tools/ab.py --build-only 'name=-DFLAG ...' ...   (here: scratch_libs/libpiko_<name>.so)
       python tools/ab.py --prebuilt CONFIG BIN scratch_libs/libpiko_a.so ...   (on the GPU box)
Each variant is compiled to /tmp and timed in its own process: median frame
time over 30 frames (L2 flushed before each, CUDA events on the draw stream)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def build(name, flags, alt=None, out_dir="/tmp"):
    import __graft_entry__ as ge
    lib = os.path.join(out_dir, f"libpiko_{name}.so")
    objs, procs = [], []
    for src, obj, extra in ge.SOURCES:  # the split translation units, compiled in parallel
        o = f"/tmp/{obj}.ab_{name}.o"
        path = alt if (alt and src == "kernels.cu") else os.path.join(ge.CSRC, src)
        procs.append(subprocess.Popen([ge._nvcc(), *ge.NVCC_FLAGS, *extra, *flags, "-I", ge.CSRC, "-c", path,
                                       "-o", o]))
        objs.append(o)
    for p in procs:
        assert p.wait() == 0
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
    r = piko.Renderer(s.W, s.H, bw, sync="async")
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream()
    ts = []
    ahead = int(os.environ.get("AB_SLEEP", "0"))  # cycles of device sleep after the flush (host runs ahead)
    for k in range(40):
        flush.fill_(float(k))
        if ahead:
            torch.cuda._sleep(ahead)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        r.draw(v, i, s.mvp, s.light, indexed=os.environ.get("AB_DRAW", "indexed") == "indexed")
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
    if sys.argv[1] == "--build-only":
        os.makedirs(os.path.join(ROOT, "scratch_libs"), exist_ok=True)
        for spec in sys.argv[2:]:
            name, _, fl = spec.partition("=")
            print(build(name, [f for f in fl.split() if f], None, os.path.join(ROOT, "scratch_libs")))
        sys.exit(0)
    if sys.argv[1] == "--prebuilt":
        cfg, bw = sys.argv[2], int(sys.argv[3])
        for rep in range(2):
            for lib in sys.argv[4:]:
                out = subprocess.run([sys.executable, __file__, "--run", lib, cfg, str(bw)], capture_output=True,
                                     text=True)
                print(f"{cfg} b{bw} {os.path.basename(lib):24s} {out.stdout.strip()} "
                      f"{out.stderr.strip()[-300:] if out.returncode else ''}", flush=True)
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
