#!/usr/bin/env python
"""Benchmark of the binned rasterizer hot path (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl piko|reference]
                    [--config c3] [--bin 16]

A step is one frame: the whole hot path (vertex transform + setup, AssignBin
count / scan / stable scatter, Schedule, per-bin raster + depth + shade +
write-back; for N > 1 also the NCCL tile-key gather and rank-0 resolve) on the
seeded synthetic scene of BASELINE.json configs[2] (1M-triangle UV sphere,
1024x768, Buddha scale) with 16x16 bins by default.  Inputs are resident in HBM;
L2 is flushed (256 MiB write) before every timed step, outside its events.
Per-step device time comes from CUDA events on the draw stream; per-kernel
times from piko_set_profiling (events between the kernels on the same stream).
N > 1: torchrun, one process per GPU, sort-first (every rank transforms all
triangles, rasterizes its bins b mod N == rank); time = max over ranks.
--impl reference times the CPU oracle (the reference arm of this tier).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Mtriangles/s at 1024x768 (binned raster frame, 1M-tri UV sphere)"
UNIT = "Mtri/s"
L2_FLUSH_BYTES = 256 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="piko", choices=["piko", "reference"])
    ap.add_argument("--config", default="c3")
    ap.add_argument("--bin", type=int, default=16)
    ap.add_argument("--cpu-budget", type=float, default=10.0, help="seconds of oracle work")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--multi", default="sort-first", choices=["sort-first", "sort-last"],
                    help="N > 1 decomposition: screen bins (sort-first) or triangle ranges + "
                         "ncclReduce(min) of the key images (sort-last)")
    ap.add_argument("--transport", default="auto", choices=["auto", "p2p", "nccl"],
                    help="sort-first tile exchange: tile kernel stores keys into rank 0's memory "
                         "over NVLink (p2p) or NCCL send/recv; auto = p2p, NCCL if any rank "
                         "cannot map the peer buffers")
    return ap.parse_args()


def workload_name(cfg, s, bw):
    return {"c2": "c2: 100 UV spheres, 100K tris", "c3": "c3: UV sphere 500x1000, 1M tris",
            "c4": "c4: random soup, 4M tris", "c5": "c5: jittered grid, 16M tris",
            "c6": "c6: Reyes, 256 bicubic patches split/diced on the device into ~1.1M micropolygon "
                  "tris"}.get(cfg, cfg) + \
        f", {s.W}x{s.H}, {bw}x{bw} bins"


class ClockSampler:
    """SM clocks and throttle reasons sampled during the run.  NVML (pynvml)
    polled every 2 ms in a thread, so even a few-millisecond timed region holds
    samples; nvidia-smi -lms 100 is the fallback when NVML is unavailable."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # NVML clocks-event-reason bits (nvml.h): sw power cap, hw slowdown, sw / hw thermal
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
            "hw_thermal_slowdown": 0x40}

    def __init__(self, gpu_index):
        self.samples = []   # (time, sm_mhz, max_mhz, [reason names])
        self.window = None
        self.proc = None
        self.stop = False
        self.source = None
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            get_reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons

            def poll():
                while not self.stop:
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        r = get_reasons(h)
                        self.samples.append((time.time(), float(sm), float(mx),
                                             [n for n, b in self.BITS.items() if r & b]))
                    except Exception:
                        pass
                    time.sleep(0.002)
            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            self.source = "nvml"
            return
        except Exception:
            pass
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            self.source = "nvidia-smi"
        except Exception:
            self.proc = None

    def _read(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

        def num(v):
            try:
                return float(v)
            except ValueError:
                return None
        for line in self.proc.stdout:
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 8 and num(f[0]) is not None:
                self.samples.append((time.time(), num(f[0]), num(f[1]),
                                     [n for n, v in zip(names, f[4:8]) if v.lower() == "active"]))

    def mark(self, t0, t1):
        self.window = (t0, t1)

    def summary(self):
        if self.source == "nvml":
            time.sleep(0.01)
            self.stop = True
        elif self.proc:
            time.sleep(0.25)
            self.proc.terminate()
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        tol = 0.0 if self.source == "nvml" else 0.15
        inwin = [x for x in self.samples if self.window and self.window[0] - tol <= x[0] <= self.window[1] + tol]
        use = inwin or self.samples
        sm = [x[1] for x in use if x[1] is not None]
        mx = [x[2] for x in use if x[2] is not None]
        reasons = sorted({n for x in use for n in x[3]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(use), "in_timed_region": bool(inwin),
                "source": self.source}


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def cpu_baseline(s, budget):
    """SURVEY 8(d) CPU oracle baseline on the GPU box's host: (i) the
    single-threaded oracle pinned to one core (sched_setaffinity, as
    `taskset -c 0`), (ii) the same source with OpenMP over row bands on all
    cores (oracle.render_mt, byte-identical frames).  Each leg renders whole
    frames of the benchmarked scene for about `budget` seconds.  Returns the
    baseline dict and the last single-threaded frame (for the parity check)."""
    import oracle
    import scenes
    patch = isinstance(s, scenes.PatchScene)

    def frame1():  # Reyes: the oracle's Split/Dice is part of the frame
        if patch:
            _, v, i = oracle.dice(s.patches, s.mvp, s.W, s.H, s.dice_px, s.max_grid)
            return oracle.render(v, i, s.mvp, s.light, s.W, s.H), i.shape[0]
        return oracle.render(s.verts, s.idx, s.mvp, s.light, s.W, s.H), s.n_tris

    def frame_mt():
        if patch:
            _, v, i = oracle.dice(s.patches, s.mvp, s.W, s.H, s.dice_px, s.max_grid)
            return oracle.render_mt(v, i, s.mvp, s.light, s.W, s.H)[1], i.shape[0]
        return oracle.render_mt(s.verts, s.idx, s.mvp, s.light, s.W, s.H)[1], s.n_tris
    aff = os.sched_getaffinity(0) if hasattr(os, "sched_getaffinity") else None
    if aff:
        os.sched_setaffinity(0, {min(aff)})
    t0 = time.perf_counter()
    frames = 0
    ref = None
    try:
        while True:
            ref, T = frame1()
            frames += 1
            if time.perf_counter() - t0 >= budget:
                break
    finally:
        if aff:
            os.sched_setaffinity(0, aff)
    dt = time.perf_counter() - t0
    out = {"value": T * frames / dt / 1e6, "unit": UNIT, "cores": 1, "kind": "oracle",
           "sample": f"{frames} full frame(s) of the benchmarked scene, single-threaded C oracle "
                     f"(gcc -O2) pinned to one core, {dt:.1f} s", "ms_per_frame": 1e3 * dt / frames,
           "cpu_model": cpu_model(), "host_cpus": os.cpu_count()}
    try:
        frame_mt()  # thread pool + pages warm
        t0 = time.perf_counter()
        mf, nthreads = 0, 0
        while True:
            nthreads, T = frame_mt()
            mf += 1
            if time.perf_counter() - t0 >= budget:
                break
        dm = time.perf_counter() - t0
        out["all_cores"] = {"value": T * mf / dm / 1e6, "unit": UNIT, "cores": nthreads,
                            "kind": "oracle (OpenMP row bands)", "ms_per_frame": 1e3 * dm / mf,
                            "sample": f"{mf} full frame(s), {dm:.1f} s, {nthreads} threads"}
    except Exception as e:  # noqa: BLE001
        out["all_cores"] = {"unavailable": str(e)}
    return out, ref


def algorithmic_bytes(stage, T, V, L, P, NB, npx, ncov, npass, cm_rows=0, cl_chunks=0):
    """Bytes the method must move per launch of a stage (
    SURVEY 8(d): 48 B per covered pixel for the winner's attributes)."""
    if stage == "vertex":     # 16 B positions in, 16 B vertex record out
        return 16 * V + 16 * V
    if stage == "setup":      # idx + vertex records in; setup records (live) + tile rects out
        if cl_chunks:         # chunk lists: the sorted pairs (4 B) instead of the rects
            return 12 * T + 16 * V + 48 * L + 4 * P
        return 12 * T + 16 * V + 48 * L + 8 * T
    if cl_chunks:             # k_cl_bins: totals, chunk bitmaps, list segments in; CSR + lists out
        return (4 * NB + 4 * NB * ((cl_chunks + 31) // 32) + 8 * P + 8 * NB) if stage == "sort" else 0
    if stage == "expand":
        if cm_rows:           # k_cm_scan: count matrix read, prefixes written, counts reset
            return 12 * cm_rows * NB + 4 * NB
        # radix pass 0: rects in, (key, primID) pairs out, bin counts
        return 8 * T + (8 * P if npass > 1 else 4 * P) + 4 * NB + (12 * NB if npass == 1 else 0)
    if stage == "sort":
        if cm_rows:           # k_cm_scatter: rects + cursor rows in, CSR values out, lists
            return 8 * T + 4 * cm_rows * NB + 4 * P + 8 * NB
        # passes >= 1: 8 B in / 8 B out (last: primIDs only) + CSR scan
        return (npass - 1) * 16 * P - 4 * P + 12 * NB if npass > 1 else 0
    if stage == "tile":       # CSR + records in; 24 B/px out; winner attributes
        return 4 * (NB + 1) + 4 * P + 48 * P + 24 * npx + 48 * ncov
    if stage == "resolve":
        return 8 * npx + 24 * npx + 48 * ncov
    return 0


def parity_check(g, s, bw, ref):
    """Compare the GPU frame of the benchmarked configuration (and its bin
    lists) with the oracle's frame of the same scene: primID and depth bits
    bit-exact, RGB within 1e-5, CSR bin lists bit-exact."""
    import numpy as np
    import oracle
    ok_p = bool(np.array_equal(g["primid"], ref["primid"]))
    ok_d = bool(np.array_equal(g["depth"].view(np.uint32), ref["depth"].view(np.uint32)))
    err = float(np.abs(g["rgba"] - ref["rgba"]).max())
    import scenes
    if isinstance(s, scenes.PatchScene):
        _, v, i = oracle.dice(s.patches, s.mvp, s.W, s.H, s.dice_px, s.max_grid)
        ost, opr = oracle.bins(v, i, s.mvp, s.W, s.H, bw, bw)
    else:
        ost, opr = oracle.bins(s.verts, s.idx, s.mvp, s.W, s.H, bw, bw)
    ok_b = bool(np.array_equal(g["bin_start"], ost) and np.array_equal(g["bin_prims"], opr))
    return {"ok": ok_p and ok_d and err <= 1e-5 and ok_b, "primid": ok_p, "depth_bits": ok_d,
            "max_rgb_err": err, "bin_lists": ok_b,
            "what": "a frame of the timed configuration (piko_draw, async) vs the CPU oracle's frame "
                    "of the same scene (cpu_baseline)"}


def run_piko(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1404_6293_b200 as piko
    import scenes

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # test hook: PIKO_BENCH_SHARE_GPU=1 puts every rank on cuda:0 with gloo for
    # torch.distributed -- exercises the N > 1 control flow (P2P transport) on a
    # one-GPU box; its timings are meaningless (ranks time-slice one GPU)
    share = os.environ.get("PIKO_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    s = scenes.make(args.config)
    patch = isinstance(s, scenes.PatchScene)  # Reyes (c6): Split/Dice on the device each frame
    bw = args.bin
    if patch:
        if world > 1:
            raise SystemExit("the Reyes config (c6) runs on one GPU")
        pt = torch.from_numpy(s.patches).to(dev)
        verts = idx = None
    else:
        verts = torch.from_numpy(s.verts).to(dev)
        idx = torch.from_numpy(s.idx).to(dev)

    def frame(indexed=False):
        if patch:
            return r.draw_patches(pt, s.mvp, s.light, s.dice_px, s.max_grid, stream)
        return r.draw(verts, idx, s.mvp, s.light, stream, indexed=indexed)
    r = piko.Renderer(s.W, s.H, bw, device=dev, sync="checked")
    transport = None
    if world > 1:
        def attach(rd, xport):
            if args.multi == "sort-last":
                piko.piko_set_multi(rd.ctx, piko.PIKO_MULTI_SORT_LAST)
            # rank 0 always broadcasts (None on failure) so no rank waits forever
            h = None
            if rank == 0:
                try:
                    h = (piko.piko_p2p_export(rd.ctx, world) if xport == "p2p"
                         else piko.piko_nccl_unique_id())
                except piko.PikoError as e:
                    print(f"rank 0: {xport} setup failed: {e}", file=sys.stderr)
            obj = [h]
            dist.broadcast_object_list(obj, src=0)
            ok = int(obj[0] is not None)
            if ok:
                try:
                    if xport == "p2p":  # CUDA IPC handles of rank 0's exchange buffers
                        if rank != 0:
                            piko.piko_p2p_import(rd.ctx, obj[0], rank, world)
                    else:
                        piko.piko_attach_comm(rd.ctx, obj[0], rank, world)
                except piko.PikoError as e:
                    print(f"rank {rank}: attach ({xport}) failed: {e}", file=sys.stderr)
                    ok = 0
            t = torch.tensor([ok], dtype=torch.int32, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MIN)  # every rank agrees on the transport
            return bool(t.item())
        transport = "nccl" if args.multi == "sort-last" or args.transport == "nccl" else "p2p"
        if not attach(r, transport):
            if args.transport != "auto" or transport == "nccl":
                raise SystemExit("multi-GPU attach failed")
            dist.barrier()  # peers unmap before rank 0 frees its exchange buffers
            if rank != 0:
                r.close()
            dist.barrier()
            if rank == 0:
                r.close()
            r = piko.Renderer(s.W, s.H, bw, device=dev)
            transport = "nccl"
            if not attach(r, transport):
                raise SystemExit("multi-GPU attach failed")
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

    # the north-star call piko_draw (no vertex count) is the headline;
    # piko_draw_indexed is timed beside it.  Warm-up in checked mode
    # (capacity settles), then the default asynchronous mode.
    indexed = False
    for _ in range(max(args.warmup, 3)):
        frame(indexed)
    piko.piko_set_sync(r.ctx, piko.PIKO_SYNC_ASYNC)
    stats = r.stats()
    ncov = int((r.primid() >= 0).sum().item()) if rank == 0 else 0

    sampler = ClockSampler(local) if rank == 0 else None
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t_wall0 = time.time()
    for k in range(args.steps):
        flush.fill_(float(k))                       # L2 flush, outside the step's events
        ev[k][0].record(stream)
        frame(indexed)
        ev[k][1].record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    t_wall1 = time.time()
    status = piko.piko_finish(r.ctx)
    if status != piko.PIKO_OK:
        raise SystemExit(f"frame status {status}: {piko.piko_last_error(r.ctx)}")
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    # second pass of K steps with per-kernel CUDA events on the draw stream
    # (the events break PDL overlap, so this pass is not the headline number)
    piko.piko_set_profiling(r.ctx, 1)
    for k in range(args.steps):
        flush.fill_(float(k))
        frame(indexed)
    torch.cuda.synchronize(dev)
    prof, nprof = piko.piko_get_profile(r.ctx)
    piko.piko_set_profiling(r.ctx, 0)
    if piko.piko_finish(r.ctx) != piko.PIKO_OK:
        raise SystemExit(f"frame status: {piko.piko_last_error(r.ctx)}")
    # the frame the parity check compares (rank 0 holds the full frame)
    gpu_frame = None
    if rank == 0 and world == 1:
        frame(indexed)
        piko.piko_finish(r.ctx)
        st_, pr_ = r.bins()
        gpu_frame = {"primid": r.primid().cpu().numpy(), "depth": r.depth.cpu().numpy().copy(),
                     "rgba": r.rgba.cpu().numpy().copy(), "bin_start": st_.cpu().numpy(),
                     "bin_prims": pr_.cpu().numpy()}
    # piko_draw_indexed (vertex count given: each vertex transformed once when
    # the mesh shares vertices), same protocol
    ie = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps if not patch else 0)]
    for _ in range(3 if not patch else 0):
        frame(True)
    torch.cuda.synchronize(dev)
    for k in range(len(ie)):
        flush.fill_(float(k))
        ie[k][0].record(stream)
        frame(True)
        ie[k][1].record(stream)
    torch.cuda.synchronize(dev)
    if piko.piko_finish(r.ctx) != piko.PIKO_OK:
        raise SystemExit(f"frame status: {piko.piko_last_error(r.ctx)}")
    idx_ms = sum(a.elapsed_time(b) for a, b in ie) if ie else float("nan")
    T = r.stats()["n_tris"] if patch else s.n_tris  # Reyes: the diced micropolygon triangles
    if world > 1:
        t = torch.tensor([idx_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        idx_ms = float(t.item())
    indexed_line = {"ms_per_step": idx_ms / args.steps, "value": T * args.steps / (idx_ms / 1e3) / 1e6,
                    "unit": UNIT, "kernels_per_frame": r.stats()["kernels_per_frame"],
                    "what": "piko_draw_indexed: vertex count given (separate once-per-vertex stage on "
                            "shared-vertex meshes)"}
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    if sampler:
        sampler.mark(t_wall0, t_wall1)

    # design alternative of sec. 7.2.1 (FreePipe: one fused kernel, no bins),
    # same protocol; reported beside the binned headline (1 GPU only)
    variants = {"piko_draw_indexed": indexed_line} if not patch else {}
    if world == 1 and not patch:
        what = {piko.PIKO_PIPE_FREEPIPE: ("freepipe", "sec. 7.2.1 FreePipe: 1 fused kernel, thread per triangle, "
                                                      "global 64-bit atomicMin + resolve; no bins"),
                piko.PIKO_PIPE_BASELINE: ("baseline", "sec. 7.1 Baseline: VS, Rasterizer, Fragment Shader, Depth "
                                                      "Test, Composite as separate kernels, fragments in HBM; no bins")}
        for pipe, (name, desc) in what.items():
            piko.piko_set_pipeline(r.ctx, pipe)
            piko.piko_set_sync(r.ctx, piko.PIKO_SYNC_CHECKED)
            for _ in range(max(args.warmup, 3)):
                frame(False)
            piko.piko_set_sync(r.ctx, piko.PIKO_SYNC_ASYNC)
            fe = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(args.steps)]
            torch.cuda.synchronize(dev)
            for k in range(args.steps):
                flush.fill_(float(k))
                fe[k][0].record(stream)
                frame(False)
                fe[k][1].record(stream)
            torch.cuda.synchronize(dev)
            fms = sum(a.elapsed_time(b) for a, b in fe) / args.steps
            variants[name] = {"ms_per_step": fms, "value": T / (fms / 1e3) / 1e6, "unit": UNIT,
                              "what": desc}
            piko.piko_finish(r.ctx)
        piko.piko_set_pipeline(r.ctx, piko.PIKO_PIPE_BINNED)
        piko.piko_set_sync(r.ctx, piko.PIKO_SYNC_CHECKED)

    # end-to-end through the public host-buffer call (H2D + frame + D2H per step)
    e2e = None
    if not args.no_e2e and not patch:
        piko.piko_set_sync(r.ctx, piko.PIKO_SYNC_CHECKED)
        hv = torch.from_numpy(s.verts).pin_memory()
        hi = torch.from_numpy(s.idx).pin_memory()
        hrgba = torch.empty((s.H, s.W, 4), dtype=torch.float32).pin_memory()
        hdepth = torch.empty((s.H, s.W), dtype=torch.float32).pin_memory()
        ke = max(3, min(args.steps, 20))
        # pipelined host-buffer calls: every step uploads its inputs and
        # downloads its frame inside the timed region; the upload of step k+1
        # overlaps the draw of k and the download of k-1 (two staging slots)
        for _ in range(3):
            piko.piko_draw_host_async(r.ctx, hv, hi, s.mvp, s.light, hrgba, hdepth, stream)
        torch.cuda.synchronize(dev)
        if piko.piko_finish(r.ctx) != 0:
            raise RuntimeError("e2e warm-up frame failed: " + piko.piko_last_error(r.ctx))
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(ke):
            piko.piko_draw_host_async(r.ctx, hv, hi, s.mvp, s.light, hrgba, hdepth, stream)
        b.record(stream)
        torch.cuda.synchronize(dev)
        if piko.piko_finish(r.ctx) != 0:  # any step's frame failed
            raise RuntimeError("e2e frame failed: " + piko.piko_last_error(r.ctx))
        e_ms = a.elapsed_time(b)
        # the synchronous call (H2D, draw, check, D2H per step) beside it
        es = []
        for _ in range(min(ke, 5)):
            a2, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a2.record(stream)
            piko.piko_draw_host(r.ctx, hv, hi, s.mvp, s.light, hrgba, hdepth, stream)
            b2.record(stream)
            torch.cuda.synchronize(dev)
            es.append(a2.elapsed_time(b2))
        if world > 1:
            t = torch.tensor([e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        e2e = {"value": T * ke / (e_ms / 1e3) / 1e6, "unit": UNIT,
               "h2d_bytes_per_step": int(hv.numel() * 4 + hi.numel() * 4),
               "d2h_bytes_per_step": int((hrgba.numel() + hdepth.numel()) * 4) if rank == 0 else 0,
               "ms_per_step": e_ms / ke, "steps": ke,
               "api": "piko_draw_host_async (pinned host buffers, 2 staging slots: H2D / draw / D2H overlapped across steps)",
               "sync_call_ms_per_step": sum(es) / len(es)}

    if rank != 0:  # peers close (unmap rank 0's P2P buffers) before rank 0 frees them
        r.close()
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    clocks = sampler.summary()
    V = piko.piko_get_diced(r.ctx)[1] if patch else s.verts.shape[0]
    P, L, NB = stats["n_pairs"], stats["n_live"], stats["n_bins"]
    npx = s.W * s.H
    per_frame = {k: v / max(nprof, 1) for k, v in prof.items()}
    cand = {k: per_frame[k] for k in ("vertex", "setup", "expand", "sort", "tile", "resolve") if per_frame[k] > 0}
    dom = max(cand, key=cand.get)
    cm_rows = stats.get("cm_rows", 0) if stats.get("assign_mode", 0) == 1 else 0
    cl_chunks = stats.get("cm_rows", 0) if stats.get("assign_mode", 0) == 2 else 0
    nb = algorithmic_bytes(dom, T, V, L, P, NB, npx, ncov, stats["radix_passes"], cm_rows, cl_chunks)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = peaks.get("hbm_gbs", 6650.0)
    achieved = nb / (per_frame[dom] / 1e3) / 1e9
    traffic = None
    tf = os.path.join(ROOT, "profiles", f"traffic_{args.config}_b{bw}.json")
    if os.path.exists(tf):
        traffic = json.load(open(tf)).get(dom)
    kname = {"vertex": "k_vertex / k_index_max", "setup": "k_setup",
             "expand": "k_cm_scan" if cm_rows else "k_radix_pass<EXPAND=true> (pass 0)",
             "sort": "k_cl_bins" if cl_chunks else "k_cm_scatter" if cm_rows else "k_radix_pass<EXPAND=false> (passes >= 1)",
             "tile": "k_tile", "resolve": "k_resolve / k_shade"}[dom]
    ncu_note = None  # the same kernel's ncu --set full counters (profiles/ncu_full_r2_<cfg>.txt)
    nf = os.path.join(ROOT, "profiles", f"ncu_full_r2_{args.config}.txt")
    if os.path.exists(nf):
        want = {"tile": "k_tile", "setup": "k_setup", "expand": "k_cm_scan" if cm_rows else "k_radix_pass",
                "sort": "k_cl_bins" if cl_chunks else "k_cm_scatter" if cm_rows else "k_radix_pass",
                "vertex": "k_vertex"}.get(dom)
        lines = [l for l in open(nf) if not l.startswith("#")]
        hdr = [l for l in open(nf) if l.startswith("# kernel")]
        for l in lines:
            if want and want in l.split(",")[0]:
                ncu_note = (hdr[0][2:].strip() if hdr else "") + " | " + l.strip()
                break
    roofline = {"bound": "hbm", "kernel": kname, "stage": dom,
                "limiter": ("latency: few resident warps per SM and dependent L2 round trips per bin "
                            "(ncu issue-active / warps-active in `ncu`)") if dom == "tile" else None,
                "ncu": ncu_note,
                "launches_per_step": max(stats["radix_passes"] - 1, 1) if (dom == "sort" and not (cm_rows or cl_chunks)) else 1,
                "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "algorithmic_bytes": nb,
                "ms_per_launch": per_frame[dom],
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6.65 TB/s"}
    frame_bytes = sum(algorithmic_bytes(k, T, V, L, P, NB, npx, ncov, stats["radix_passes"], cm_rows, cl_chunks)
                      for k in ("vertex", "setup", "expand", "sort", "tile") if per_frame.get(k, 0) > 0.004)
    # BASELINE.md's frame metric: ncu-measured DRAM bytes of one whole frame
    # (range replay: all kernels in one range, L2 write-backs included --
    # tools/frame_dram.py); else the sum of per-kernel cold replays
    measured, measured_note = None, None
    ff = os.path.join(ROOT, "profiles", f"traffic_frame_{args.config}_b{bw}.json")
    if os.path.exists(ff):
        fj = json.load(open(ff))
        measured = int(fj["frame_bytes"])
        measured_note = f"profiles/traffic_frame_{args.config}_b{bw}.json: " + fj.get("_note", "")
    elif os.path.exists(tf):
        tj = json.load(open(tf))
        ran = [k for k in ("vertex", "setup", "expand", "sort", "tile") if per_frame.get(k, 0) > 0.004]
        if all(k in tj for k in ran):
            measured = int(sum(tj[k] for k in ran))
            measured_note = ("sum of ncu dram__bytes_read+write per kernel of one frame "
                             "(profiles/traffic_*.json; ncu replays each kernel cold)")
    ms = total_ms / args.steps
    out = {
        "metric": METRIC, "value": T * args.steps / (total_ms / 1e3) / 1e6, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f32+int32/int64", "data": "synthetic (seeded scenes/)",
        "config": {"workload": workload_name(args.config, s, bw), "config": args.config,
                   "width": s.W, "height": s.H, "bin": bw, "n_tris": T, "n_verts": V,
                   "n_pairs": P, "n_live": L, "covered_px": ncov, "l2": "flushed (256 MiB) before every step",
                   "assign": ("chunk lists" if cl_chunks else "count matrix" if cm_rows
                              else f"radix x{stats['radix_passes']}"),
                   "parallelism": f"{args.multi} x{world} ({transport})" if world > 1 else "1 GPU"},
        "fps": 1e3 / ms,
        "ms_p10_p50_p90": [float(x) for x in np.percentile(step_ms, [10, 50, 90])],
        "frame_roofline": {"algorithmic_bytes": frame_bytes, "frac": frame_bytes / (ms / 1e3) / 1e9 / peak,
                           "measured_bytes": measured,
                           "frac_measured": measured / (ms / 1e3) / 1e9 / peak if measured else None,
                           "measured_note": measured_note},
        "kernel_ms": per_frame,
        # every stage against the same HBM peak (algorithmic bytes per launch /
        # its event time) -- the dominant one is `roofline`
        "stage_roofline": {k: {"ms": per_frame[k],
                               "algorithmic_bytes": algorithmic_bytes(k, T, V, L, P, NB, npx, ncov, stats["radix_passes"],
                                                                      cm_rows, cl_chunks),
                               "frac": algorithmic_bytes(k, T, V, L, P, NB, npx, ncov, stats["radix_passes"], cm_rows,
                                                         cl_chunks) / (per_frame[k] / 1e3) / 1e9 / peak}
                           for k in ("vertex", "setup", "expand", "sort", "tile") if per_frame.get(k, 0) > 0.004},
        "kernel_ms_note": "per-stage CUDA-event times from a second K-step pass (events between kernels)",
        "api": "piko_draw (north-star C ABI call via ctypes, PIKO_SYNC_ASYNC)",
        "roofline": roofline,
        "variants": variants,
        "gpu_launches": stats["kernels_per_frame"] * args.steps,
        "clocks": clocks,
        "e2e": e2e,
    }
    if world == 1 and not args.no_cpu:
        out["cpu_baseline"], ref = cpu_baseline(s, args.cpu_budget)
        out["parity"] = parity_check(gpu_frame, s, bw, ref)
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    r.close()


def run_reference(args):
    """Reference arm = the CPU oracle as it stands, on rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    import scenes
    s = scenes.make(args.config)
    for _ in range(args.warmup):
        oracle.render(s.verts, s.idx, s.mvp, s.light, s.W, s.H)
    t = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.render(s.verts, s.idx, s.mvp, s.light, s.W, s.H)
        t.append(time.perf_counter() - t0)
    total = sum(t)
    v = s.n_tris * args.steps / total / 1e6
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT,
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f32+int32/int64", "data": "synthetic (seeded scenes/)",
           "config": {"workload": workload_name(args.config, s, args.bin), "config": args.config,
                      "width": s.W, "height": s.H, "bin": args.bin, "n_tris": s.n_tris},
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                            "sample": f"{args.steps} full frames, single-threaded C oracle (gcc -O2)"},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_piko(a)
