#!/usr/bin/env python
"""Per-CTA phase timelines (globaltimer ns) of the count-matrix AssignBin
kernels: builds a -DPIKO_K1_TIMING libpiko, renders frames, prints phases."""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as ge

extra = [f for f in os.environ.get("PIKO_EXP", "").split() if f]
lib = f"/tmp/libpiko_cmt{os.getpid()}.so"
objs = []
for src in sorted({src for src, _, _ in ge.SOURCES}):
    o = f"/tmp/{src}.cmt.o"
    subprocess.check_call([ge._nvcc(), *ge.NVCC_FLAGS, "-DPIKO_K1_TIMING", *extra, "-c", os.path.join(ge.CSRC, src), "-o", o])
    objs.append(o)
subprocess.check_call([ge._nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", lib, "-ldl", "-lcudart"])
import paper_1404_6293_b200 as piko  # noqa: E402
piko.LIB_PATH = lib
piko._lib = piko.lib = piko._load()
import numpy as np  # noqa: E402
import torch  # noqa: E402
import scenes  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
s = scenes.make(cfg)
v = torch.from_numpy(s.verts).cuda()
i = torch.from_numpy(s.idx).cuda()
r = piko.Renderer(s.W, s.H, 16)
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
h = ctypes.CDLL(lib)
piko.piko_set_sync(r.ctx, piko.PIKO_SYNC_ASYNC)
st = torch.cuda.current_stream()
for k in range(4):
    if not os.environ.get("TL_NOFLUSH"):
        flush.fill_(float(k))
    if k == 3:  # reset the vertex-start slots (atomicMin/Max) before the measured frame
        z = np.zeros((4, 8192, 8), np.uint64)
        z[0, 8190, 0] = z[0, 8191, 0] = np.uint64(2**63)
        torch.cuda.synchronize()
        h.piko_dbg_k1_set(z.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(z.nbytes))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    r.draw(v, i, s.mvp, s.light)
    e1.record(st)
    torch.cuda.synchronize()
print(f"event-timed frame: {e0.elapsed_time(e1) * 1000:.1f} us")
piko.piko_finish(r.ctx)
buf = np.zeros((4, 8192, 8), np.uint64)
assert h.piko_dbg_k1_times(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes)) == 0
T0 = int(buf[0, 0, 0])
vs = buf[0, 8190].astype(np.int64)
print(f"k_vertex: first CTA start {int(vs[0]) - T0} ns, last CTA start {int(vs[1]) - T0}, first past wait {int(buf[0, 8191, 0]) - T0} (rel. k_setup chunk 0)")
n1 = (s.n_tris + 1023) // 1024
kk = buf[0, :n1].astype(np.int64) - T0
print(f"k_setup: CTAs {n1}, start..end {kk[:,0].min()}..{kk[:,5].max()}, start p50 {np.median(kk[:,0]):.0f}; "
      f"loads {np.median(kk[:,1]-kk[:,0]):.0f} setup {np.median(kk[:,2]-kk[:,1]):.0f} rest {np.median(kk[:,5]-kk[:,2]):.0f}")
def rows(k, n):
    t = buf[k, :n].astype(np.int64)
    return t[t[:, 0] > T0] - T0
cs = rows(1, 8000)
last = cs[cs[:, 3] > 0]
print(f"k_cm_scan: CTAs {len(cs)}, start {cs[:,0].min()}..{cs[:,0].max()}, sweeps end max {cs[:,2].max()}; "
      f"sweep1 {np.median(cs[:,1]-cs[:,0]):.0f} (p90 {np.percentile(cs[:,1]-cs[:,0],90):.0f}), "
      f"sweep2 {np.median(cs[:,2]-cs[:,1]):.0f}; last CTA bin scan end {last[:,3].max() if len(last) else -1}")
sc = rows(2, 8000)
print(f"k_cm_scatter: CTAs {len(sc)}, start {sc[:,0].min()}..{sc[:,0].max()} (p50 {np.median(sc[:,0]):.0f}), "
      f"pdl-wait done {sc[:,1].min()}..{sc[:,1].max()}")
names = {1: "pdl wait done", 3: "counts+offsets", 4: "expanded", 5: "digits+cursors", 6: "ranked+written", 2: "end"}
for k in (1, 3, 4, 5, 6, 2):
    m = sc[:, k] > 0
    if m.any():
        print(f"   {names[k]:16s}: {m.sum()} CTAs, time p50 {np.median(sc[m,k]):.0f} (min {sc[m,k].min()}, max {sc[m,k].max()})")
u = buf[2, :8000, 7].astype(np.int64)
u = u[u > 0]
if len(u):
    print(f"   U (touched bins per window): p50 {np.median(u):.0f} max {u.max()}")
t = buf[3, :8192].astype(np.int64)
t = t[(t[:, 0] > T0) & (t[:, 2] >= t[:, 0])] - T0
print(f"k_tile bins: first start {t[:,0].min()}, last end {t[:,2].max()}")
st = r.stats()
nb = st["owned_bins"]
t = buf[3, :min(nb, 8192)].astype(np.int64)
t = t[(t[:, 0] > T0) & (t[:, 2] >= t[:, 0])]
base = t[:, 0].min()
ne = t[:, 3]
for lo, hi in ((0, 0), (1, 64), (65, 256), (257, 1024), (1025, 1 << 30)):
    m = (ne >= lo) & (ne <= hi)
    if m.any():
        r1 = t[m, 1] - t[m, 0]
        r2 = t[m, 2] - t[m, 1]
        print(f"   bins with {lo}-{hi} pairs: {m.sum():5d}  raster median {np.median(r1):7.0f} p90 {np.percentile(r1,90):7.0f}"
              f"  writeback median {np.median(r2):7.0f} p90 {np.percentile(r2,90):7.0f}")
m = (ne >= 257)
if m.any():
    tm = t[m]
    print(f"   heavy bins phases (median ns): clear {np.median(tm[:,5]-tm[:,0]):.0f}  rounds {np.median(tm[:,6]-tm[:,5]):.0f}"
          f"  wait+sync {np.median(tm[:,7]-tm[:,6]):.0f}  prologue+drain {np.median(tm[:,1]-tm[:,7]):.0f}  writeback {np.median(tm[:,2]-tm[:,1]):.0f}")
if m.any():  # the same phases for each CTA's first heavy item vs its later ones
    tm = t[m]
    first = np.zeros(len(tm), bool)
    seen = set()
    for j in np.argsort(tm[:, 0]):
        c_ = int(tm[j, 4])
        if c_ not in seen:
            seen.add(c_)
            first[j] = True
    for nm, sel in (("first", first), ("later", ~first)):
        if sel.any():
            u = tm[sel]
            print(f"   heavy {nm:5s} items ({sel.sum()}): pairs {np.median(u[:,3]):.0f} clear {np.median(u[:,5]-u[:,0]):.0f}"
                  f"  rounds {np.median(u[:,6]-u[:,5]):.0f}  wait+sync {np.median(u[:,7]-u[:,6]):.0f}"
                  f"  prologue+drain {np.median(u[:,1]-u[:,7]):.0f}  writeback {np.median(u[:,2]-u[:,1]):.0f}")
cta = t[:, 4]
per = np.bincount(cta.astype(np.int64))
print(f"   bins per CTA: min {per[per>0].min()} max {per.max()} CTAs {np.count_nonzero(per)}")
c = buf[0, 7000:7000 + 1024].astype(np.int64)
c = c[c[:, 0] > T0] - T0
print(f"   k_tile CTAs: resident first {c[:,3].min()} p50 {np.median(c[:,3]):.0f}; past pdl wait {c[:,0].min()}..{c[:,0].max()};"
      f" bin loop end p50 {np.median(c[:,1]):.0f} max {c[:,1].max()}; CTA end p50 {np.median(c[:,2]):.0f} max {c[:,2].max()}")
tt = buf[3, :min(nb, 8192)].astype(np.int64)
ok = (tt[:, 0] > T0) & (tt[:, 2] >= tt[:, 0])
rows = [(int(tt[b, 4]), b, int(tt[b, 3]), tt[b, 0] - T0, tt[b, 1] - tt[b, 0], tt[b, 2] - tt[b, 1])
        for b in np.nonzero(ok)[0]]
by = {}
for cta, b, n, st_, ra, wb in rows:
    by.setdefault(cta, []).append((st_, b, n, ra, wb))
ends = sorted(((max(s_ + r_ + w_ for s_, _, _, r_, w_ in v), c) for c, v in by.items()), reverse=True)
print("   slowest CTAs (end ns): bins as (start, pairs, raster, writeback)")
for e_, cc in ends[:6]:
    print(f"     cta {cc:4d} end {e_:6d}: " + "  ".join(f"({s_},{n},{r_},{w_})" for s_, _, n, r_, w_ in sorted(by[cc])))
firsts = sorted(v[0][0] for v in (sorted(x) for x in by.values()))
print(f"   first-bin start across CTAs: min {firsts[0]} p50 {np.median(firsts):.0f} max {max(firsts)}")
seconds = sorted(sorted(x)[1][0] for x in by.values() if len(x) > 1)
if seconds:
    print(f"   second-bin start: min {seconds[0]} p50 {np.median(seconds):.0f} max {max(seconds)}; CTAs with 2+ bins {len(seconds)}")
