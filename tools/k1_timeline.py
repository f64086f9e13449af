#!/usr/bin/env python
"""Build a -DPIKO_K1_TIMING variant of libpiko, render frames and print the
per-CTA phase timelines (globaltimer ns) of k_setup, the radix passes and k_tile."""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as ge

extra = [f for f in os.environ.get("PIKO_EXP", "").split() if f]
lib = f"/tmp/libpiko_timing{os.getpid()}.so"
objs = []
for src in sorted({src for src, _, _ in ge.SOURCES}):  # one TU per source (no tile split)
    o = f"/tmp/{src}.timing.o"
    subprocess.check_call([ge._nvcc(), *ge.NVCC_FLAGS, "-DPIKO_K1_TIMING", *extra, "-c",
                           os.path.join(ge.CSRC, src), "-o", o])
    objs.append(o)
subprocess.check_call([ge._nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs,
                       "-o", lib, "-ldl", "-lcudart"])
import paper_1404_6293_b200 as piko  # noqa: E402
piko.LIB_PATH = lib
piko._lib = piko.lib = piko._load()
import numpy as np  # noqa: E402
import torch  # noqa: E402

import scenes  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
bw = int(sys.argv[2]) if len(sys.argv) > 2 else 16
s = scenes.make(cfg)
v = torch.from_numpy(s.verts).cuda()
i = torch.from_numpy(s.idx).cuda()
r = piko.Renderer(s.W, s.H, bw)
for _ in range(3):
    r.draw(v, i, s.mvp, s.light)
torch.cuda.synchronize()
st = r.stats()
buf = np.zeros((4, 8192, 8), np.uint64)
h = ctypes.CDLL(lib)
rc = h.piko_dbg_k1_times(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes))
assert rc == 0, rc
T0 = int(buf[0, 0, 0])


def show(name, t, phases, n):
    t = t[:n].astype(np.int64)
    ok = t[:, 0] > 0
    t = t[ok]
    base = t[:, 0].min()
    print(f"== {name}: {len(t)} units, start {base - T0} ns after k_setup chunk 0, span {t[:, len(phases)-1].max() - base} ns")
    for k in range(1, len(phases)):
        d = t[:, k] - t[:, k - 1]
        print(f"   {phases[k]:16s} median {np.median(d):8.0f}  p90 {np.percentile(d, 90):8.0f}  max {d.max():8.0f}")
    srt = np.sort(t[:, 0] - base)
    print(f"   unit start: p50 {srt[len(srt)//2]}  last {srt[-1]};  unit end p50 {np.median(t[:, len(phases)-1]-base):.0f}")


n1 = (s.n_tris + 1023) // 1024
kk = buf[0, :n1].astype(np.int64)
kk = kk[kk[:, 0] > 0]
b0 = kk[:, 0].min()
print(f"== k_setup: {len(kk)} CTAs, span {kk[:, 5].max() - b0} ns; loads median {np.median(kk[:,1]-kk[:,0]):.0f}, "
      f"setup median {np.median(kk[:,2]-kk[:,1]):.0f}, hist median {np.median(kk[:,5]-kk[:,2]):.0f}")
nrx0 = int((buf[1, :8000, 0] > 0).sum())
show("radix pass 0 (expand)", buf[1], ["start", "expand", "rank", "lookback", "scatter"], nrx0)
e = buf[1, :nrx0].astype(np.int64)
print("   expand detail: loads+counts median %.0f, scan %.0f, expansion %.0f, reload %.0f" % (
    np.median(e[:, 5] - e[:, 0]), np.median(e[:, 6] - e[:, 5]), np.median(e[:, 7] - e[:, 6]),
    np.median(e[:, 1] - e[:, 7])))
lb = np.zeros((2, 8192, 8), np.uint64)
if h.piko_dbg_rx_lb(lb.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(lb.nbytes)) == 0:
    for p_, n_ in ((0, nrx0), (1, int((buf[2, :8000, 0] > 0).sum()))):
        tt = buf[1 + p_, :n_].astype(np.int64)
        ll = lb[p_, :n_].astype(np.int64)
        ok = (tt[:, 2] > 0) & (ll[:, 0] > 0)
        l1 = ll[ok, 0] - tt[ok, 2]
        l2 = tt[ok, 3] - ll[ok, 0]
        print(f"   pass {p_} look-back: level-1 median {np.median(l1):.0f} p90 {np.percentile(l1, 90):.0f};"
              f" level-2 median {np.median(l2):.0f} p90 {np.percentile(l2, 90):.0f};"
              f" probes l1 median {np.median(ll[ok, 1]):.0f} max {ll[ok, 1].max()},"
              f" l2 median {np.median(ll[ok, 2]):.0f} max {ll[ok, 2].max()}")
        ga = ll[:, 3]
        gm = (ga > 0) & (tt[:, 0] > 0) & (ga > tt[:, 0])
        if gm.any():
            # group aggregate published vs the arriving chunk's expand end
            d = ga[gm] - tt[gm, 1]
            print(f"   pass {p_} group aggregate publish after own expand/load end: median {np.median(d):.0f} p90 {np.percentile(d, 90):.0f}")
            a1 = ll[gm, 4] - tt[gm, 1]
            a2 = ll[gm, 5] - ll[gm, 4]
            a3 = ll[gm, 3] - ll[gm, 5]
            print(f"      -> arrival atomic done {np.median(a1):.0f} (p90 {np.percentile(a1, 90):.0f}),"
                  f" group loads {np.median(a2):.0f} (p90 {np.percentile(a2, 90):.0f}),"
                  f" read-check-store {np.median(a3):.0f} (p90 {np.percentile(a3, 90):.0f})")
nrx = int((buf[2, :8000, 0] > 0).sum())
show("radix pass 1", buf[2], ["start", "load", "rank", "lookback", "scatter"], nrx)
nb = st["owned_bins"]
t = buf[3, :min(nb, 8192)].astype(np.int64)
t = t[(t[:, 0] > T0) & (t[:, 2] >= t[:, 0])]   # bins recorded in this frame
base = t[:, 0].min()
print(f"== k_tile: {len(t)} bins recorded, first bin start {base - T0} ns after k_setup chunk 0, "
      f"last bin end {t[:, 2].max() - T0} ns")
ne = t[:, 3]
for lo, hi in ((0, 0), (1, 256), (257, 1024), (1025, 1 << 30)):
    m = (ne >= lo) & (ne <= hi)
    if m.any():
        r1 = t[m, 1] - t[m, 0]
        r2 = t[m, 2] - t[m, 1]
        print(f"   bins with {lo}-{hi} pairs: {m.sum():5d}  raster median {np.median(r1):7.0f} p90 {np.percentile(r1,90):7.0f}"
              f"  writeback median {np.median(r2):7.0f} p90 {np.percentile(r2,90):7.0f}")
cta = t[:, 4]
per = np.bincount(cta.astype(np.int64))
busy = np.zeros(per.size)
for c in range(per.size):
    m = cta == c
    if m.any():
        busy[c] = (t[m, 2] - t[m, 0]).sum()
print(f"   bins per CTA: min {per[per>0].min()} max {per.max()};  CTA busy ns: median {np.median(busy[busy>0]):.0f} max {busy.max():.0f}")
print(f"   frame timeline (ns after k_setup chunk 0): expand {int(buf[1, :nrx0, 0].astype(np.int64).min() - T0)}"
      f"..{int(buf[1, :nrx0, 4].astype(np.int64).max() - T0)}, sort "
      f"{int(buf[2, :nrx, 0][buf[2, :nrx, 0] > 0].astype(np.int64).min() - T0)}.."
      f"{int(buf[2, :nrx, 4].astype(np.int64).max() - T0)}, tile {base - T0}..{t[:, 2].max() - T0}")

c = buf[0, 7000:7000 + 1024].astype(np.int64)
c = c[c[:, 0] > T0]
b0 = c[:, 0].min()
print(f"   k_tile CTAs first start {b0 - T0} ns after k_setup chunk 0")
print(f"== k_tile per CTA ({len(c)} CTAs): start spread {c[:,0].max()-b0} ns; resident (before griddepcontrol.wait):"
      f" first {c[:,3].min()-T0} p50 {int(np.median(c[:,3]))-T0} last {c[:,3].max()-T0} ns after k_setup chunk 0")
for p_ in (0, 1):
    sc = buf[1 + p_, 8100:8164].astype(np.int64)
    sc = sc[sc[:, 0] > T0]
    if len(sc):
        print(f"   bin-scan tiles in radix pass {p_}: {len(sc)}, start {sc[:,0].min()-T0}..{sc[:,0].max()-T0}, end max {sc[:,1].max()-T0} ns")
        for r_ in sc:
            print("      tile: start %d  +load/scan %d  +lookback %d  +kinds %d  +atomics %d  +stores %d" % (
                r_[0] - T0, r_[2] - r_[0], r_[3] - r_[2], r_[4] - r_[3], r_[5] - r_[4], r_[1] - r_[5]))
print(f"   work-list phase end: median {np.median(c[:,1]-b0):.0f} p90 {np.percentile(c[:,1]-b0,90):.0f} max {(c[:,1]-b0).max()}")
print(f"   CTA end:             median {np.median(c[:,2]-b0):.0f} p90 {np.percentile(c[:,2]-b0,90):.0f} max {(c[:,2]-b0).max()}")

# slowest CTAs: the bins they processed (pairs, start/raster/writeback ns relative to the first bin)
tt = buf[3, :min(nb, 8192)].astype(np.int64)
ok = (tt[:, 0] > T0) & (tt[:, 2] >= tt[:, 0])
rows = [(int(tt[b, 4]), b, int(tt[b, 3]), tt[b, 0] - base, tt[b, 1] - tt[b, 0], tt[b, 2] - tt[b, 1])
        for b in np.nonzero(ok)[0]]
by = {}
for cta, b, n, st_, ra, wb in rows:
    by.setdefault(cta, []).append((st_, b, n, ra, wb))
ends = sorted(((max(s_ + r_ + w_ for s_, _, _, r_, w_ in v), c) for c, v in by.items()), reverse=True)
print("   slowest CTAs (end ns): bins as (start, pairs, raster, writeback)")
for e_, c in ends[:8]:
    print(f"     cta {c:4d} end {e_:6d}: " + "  ".join(f"({s_},{n},{r_},{w_})" for s_, _, n, r_, w_ in sorted(by[c])))
firsts = sorted(v[0][0] for v in (sorted(x) for x in by.values()))
print(f"   first-bin start across CTAs: p50 {np.median(firsts):.0f} max {max(firsts)}")
pairs_sorted = sorted((n for _, _, n, _, _, _ in rows), reverse=True)
print(f"   pair counts: top {pairs_sorted[:5]}, #bins {len(rows)}, sum {sum(pairs_sorted)}")
