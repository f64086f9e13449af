"""Sort-first multi-GPU path (DirectMap round robin P:688).

* CPU (gloo, world_size 2): the exchange protocol -- every rank packs the keys
  of the bins it owns (library's host-only plan, piko_owned_bins) in payload
  order, rank 0 gathers rank-major and unpacks with the resolve kernel's
  indexing; the reassembled key image equals the oracle's.
* GPU: the device data path on one GPU -- per-rank packed tile keys from the
  tile kernel (piko_draw_tile_keys), concatenated rank-major, resolved by the
  rank-0 kernel (piko_resolve_keys) == the oracle frame, bit-exact.  (NCCL
  itself needs one GPU per rank; the transport is a byte copy of these buffers.)
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

import scenes

W, H, BW = 200, 120, 16


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _pack(keys_img, owned, bw, bh, binsX):
    out = np.full((len(owned), bw * bh), np.uint64(0xFFFFFFFFFFFFFFFF), np.uint64)
    for k, b in enumerate(owned):
        by, bx = divmod(int(b), binsX)
        tile = keys_img[by * bh:(by + 1) * bh, bx * bw:(bx + 1) * bw]
        out[k].reshape(bh, bw)[:tile.shape[0], :tile.shape[1]] = tile
    return out


def _unpack(all_keys, R, owned_max, bw, bh, W_, H_):
    """k_resolve's indexing: pixel -> bin b -> rank b % R, slot b // R."""
    binsX = -(-W_ // bw)
    img = np.empty((H_, W_), np.uint64)
    for y in range(H_):
        for x in range(W_):
            b = (y // bh) * binsX + x // bw
            img[y, x] = all_keys[b % R, b // R, (y % bh) * bw + (x % bw)]
    return img


def _gloo_worker(rank, world, port, keys_img, result):
    import torch
    import torch.distributed as dist
    import paper_1404_6293_b200 as piko
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    binsX = -(-W // BW)
    owned = piko.piko_owned_bins(W, H, BW, BW, rank, world)
    owned_max = len(piko.piko_owned_bins(W, H, BW, BW, 0, world))
    payload = np.full((owned_max, BW * BW), np.uint64(0xFFFFFFFFFFFFFFFF), np.uint64)
    payload[:len(owned)] = _pack(keys_img, owned, BW, BW, binsX)
    t = torch.from_numpy(payload.view(np.int64))
    gathered = [torch.empty_like(t) for _ in range(world)] if rank == 0 else None
    dist.gather(t, gathered, dst=0)
    if rank == 0:
        all_keys = np.stack([g.numpy().view(np.uint64) for g in gathered])
        result["img"] = _unpack(all_keys, world, owned_max, BW, BW, W, H)
    dist.destroy_process_group()


def test_owned_bins_partition():
    import paper_1404_6293_b200 as piko
    NB = (-(-W // BW)) * (-(-H // BW))
    for R in (1, 2, 3, 4, 8):
        seen = np.concatenate([piko.piko_owned_bins(W, H, BW, BW, r, R) for r in range(R)])
        assert sorted(seen.tolist()) == list(range(NB))


def test_gloo_exchange_reassembles_frame(oracle_lib):
    import multiprocessing as mp
    import threading
    s = scenes.scene_soup(4000, W, H, seed=71, name="soup")
    keys = oracle_lib.render(s.verts, s.idx, s.mvp, s.light, W, H, want_keys=True)["keys"]
    port = _free_port()
    result = {}
    # rank 1 in a subprocess, rank 0 in this process
    ctx = mp.get_context("spawn")
    p = ctx.Process(target=_gloo_worker, args=(1, 2, port, keys, {}))
    p.start()
    _gloo_worker(0, 2, port, keys, result)
    p.join(timeout=120)
    assert p.exitcode == 0
    assert np.array_equal(result["img"], keys)


@pytest.mark.gpu
@pytest.mark.parametrize("R", [2, 3, 4])
def test_gpu_tile_keys_gather_resolve(oracle_lib, R):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    import paper_1404_6293_b200 as piko
    s = scenes.scene_c2()
    dev = torch.device("cuda:0")
    v = torch.from_numpy(s.verts).to(dev)
    i = torch.from_numpy(s.idx).to(dev)
    renderers = [piko.Renderer(s.W, s.H, 16, device=dev) for _ in range(R)]
    for r, rd in enumerate(renderers):
        piko.piko_set_partition(rd.ctx, r, R)
    n = piko.piko_tile_keys_count(renderers[0].ctx)
    all_keys = torch.empty((R, n), dtype=torch.int64, device=dev)
    for r, rd in enumerate(renderers):
        piko.piko_draw_tile_keys(rd.ctx, v, i, s.mvp, s.light, all_keys[r])
    r0 = renderers[0]
    piko.piko_resolve_keys(r0.ctx, v, i, s.mvp, s.light, R, all_keys, r0.rgba, r0.depth)
    torch.cuda.synchronize()
    ref = oracle_lib.render(s.verts, s.idx, s.mvp, s.light, s.W, s.H)
    assert np.array_equal(r0.primid().cpu().numpy(), ref["primid"])
    assert np.array_equal(r0.depth.cpu().numpy().view(np.uint32), ref["depth"].view(np.uint32))
    assert np.abs(r0.rgba.cpu().numpy() - ref["rgba"]).max() <= 1e-5
    # the gathered payload itself: every pixel's key is the oracle's
    keys = oracle_lib.render(s.verts, s.idx, s.mvp, s.light, s.W, s.H, want_keys=True)["keys"]
    owned_max = n // (16 * 16)
    img = _unpack(all_keys.cpu().numpy().view(np.uint64).reshape(R, owned_max, 256), R, owned_max,
                  16, 16, s.W, s.H)
    assert np.array_equal(img, keys)
    for rd in renderers:
        rd.close()


@pytest.mark.gpu
@pytest.mark.parametrize("R", [2, 3, 4])
def test_gpu_p2p_transport_virtual_ranks(oracle_lib, R):
    """P2P transport (tile kernel stores keys straight into rank 0's buffer,
    arrival flags, rank-0 resolve waits): virtual ranks sharing rank 0's
    buffers on one device, several frames with alternating views so a wrong
    slot parity or a stale key image fails."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    import paper_1404_6293_b200 as piko
    s = scenes.scene_c2()
    dev = torch.device("cuda:0")
    v = torch.from_numpy(s.verts).to(dev)
    i = torch.from_numpy(s.idx).to(dev)
    rds = [piko.Renderer(s.W, s.H, 16, device=dev) for _ in range(R)]
    piko.piko_attach_local_peers(rds[0].ctx, rds[0].ctx, 0, R)
    for r in range(1, R):
        piko.piko_attach_local_peers(rds[r].ctx, rds[0].ctx, r, R)
    views = [s.mvp, scenes.perspective_mvp(fovy_deg=50.0)]  # two views: different keys
    refs = [oracle_lib.render(s.verts, s.idx, mv, s.light, s.W, s.H) for mv in views]
    for f in range(5):
        mv = views[f % 2]
        for r in list(range(1, R)) + [0]:
            rds[r].draw(v, i, mv, s.light)
        torch.cuda.synchronize()
        ref = refs[f % 2]
        r0 = rds[0]
        assert np.array_equal(r0.primid().cpu().numpy(), ref["primid"]), f"frame {f}"
        assert np.array_equal(r0.depth.cpu().numpy().view(np.uint32), ref["depth"].view(np.uint32))
        assert np.abs(r0.rgba.cpu().numpy() - ref["rgba"]).max() <= 1e-5
    for rd in rds[1:] + rds[:1]:
        rd.close()


def _p2p_ipc_worker(rank, world, port, result):
    """One process of the two-process P2P test (both on cuda:0): CUDA IPC
    handles travel over gloo, then every frame rank 1's tile kernel stores its
    keys into rank 0's buffer and raises its flag; rank 0 resolves."""
    import torch
    import torch.distributed as dist
    import paper_1404_6293_b200 as piko
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    s = scenes.scene_soup(20000, 333, 200, seed=91, name="soup")
    dev = torch.device("cuda:0")
    v = torch.from_numpy(s.verts).to(dev)
    i = torch.from_numpy(s.idx).to(dev)
    r = piko.Renderer(s.W, s.H, 16, device=dev)
    obj = [piko.piko_p2p_export(r.ctx, world) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    if rank != 0:
        piko.piko_p2p_import(r.ctx, obj[0], rank, world)
    dist.barrier()  # every rank mapped and ready before the first frame
    views = [s.mvp, np.array([[0.9, 0.1, 0, 0.05], [-0.1, 0.9, 0, 0], [0, 0, 1, 0], [0, 0, 0, 1]],
                             np.float32).reshape(16)]
    frames = []
    for f in range(4):
        r.draw(v, i, views[f % 2], s.light)
        torch.cuda.synchronize()
        if rank == 0:
            frames.append((r.primid().cpu().numpy(), r.depth.cpu().numpy().copy(),
                           r.rgba.cpu().numpy().copy()))
    dist.barrier()  # rank 0's buffers outlive the peers' mappings
    if rank != 0:
        r.close()
    dist.barrier()
    if rank == 0:
        r.close()
        result["frames"] = frames
        result["scene"] = s
        result["views"] = views
    dist.destroy_process_group()


@pytest.mark.gpu
def test_gpu_p2p_transport_two_processes(oracle_lib):
    """The cross-process part of the P2P transport (CUDA IPC handle export /
    import, system-scope flags between processes) on one device: rank 0 in this
    process, rank 1 in a spawned one; rank 0's frames == oracle, bit-exact."""
    import multiprocessing as mp
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    port = _free_port()
    result = {}
    ctx = mp.get_context("spawn")
    p = ctx.Process(target=_p2p_ipc_worker, args=(1, 2, port, {}))
    p.start()
    _p2p_ipc_worker(0, 2, port, result)
    p.join(timeout=300)
    assert p.exitcode == 0
    s = result["scene"]
    for f, (prim, depth, rgba) in enumerate(result["frames"]):
        ref = oracle_lib.render(s.verts, s.idx, result["views"][f % 2], s.light, s.W, s.H)
        assert np.array_equal(prim, ref["primid"]), f"frame {f}"
        assert np.array_equal(depth.view(np.uint32), ref["depth"].view(np.uint32)), f"frame {f}"
        assert np.abs(rgba - ref["rgba"]).max() <= 1e-5


@pytest.mark.gpu
def test_gpu_peer_overflow_reaches_rank0(oracle_lib):
    """A rank whose pair capacity overflows sends empty bins; its status word
    travels with its keys (P2P: next to its arrival flag, by slot parity), so
    rank 0 reports PIKO_ECAPACITY for that frame too instead of returning a
    frame with holes.  Scene: 300 tall thin triangles inside odd 8-px bin
    columns only (binsX = 128 is even, so with R = 2 every pair belongs to
    rank 1: 28800 pairs against an initial capacity of ~10^4)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    import paper_1404_6293_b200 as piko
    from tests.helpers import pixel_scene
    R = 2
    tris, zs = [], []
    for k in range(300):
        tx = 2 * (k % 64) + 1
        tris.append([(8 * tx + 1.0, 0.0), (8 * tx + 7.0, 0.0), (8 * tx + 4.0, 767.0)])
        zs.append(0.1 + 0.8 * k / 300)
    v, i, m = pixel_scene(tris, np.array(zs), 1024, 768)
    s = scenes.Scene("odd", 1024, 768, (8,), v, i, m)
    dev = torch.device("cuda:0")
    vt, it = torch.from_numpy(v).to(dev), torch.from_numpy(i).to(dev)
    rds = [piko.Renderer(s.W, s.H, 8, device=dev) for _ in range(R)]
    piko.piko_attach_local_peers(rds[0].ctx, rds[0].ctx, 0, R)
    for r in range(1, R):
        piko.piko_attach_local_peers(rds[r].ctx, rds[0].ctx, r, R)
    ref = oracle_lib.render(s.verts, s.idx, s.mvp, s.light, s.W, s.H)
    try:
        for f in range(3):
            rcs = {r: rds[r].draw(vt, it, m, s.light, check=False) for r in list(range(1, R)) + [0]}
            torch.cuda.synchronize()
            if f == 0:  # rank 1 holds every pair: it overflows, and rank 0 must say so
                assert rcs[1] == piko.PIKO_ECAPACITY
                assert rcs[0] == piko.PIKO_ECAPACITY, piko.piko_last_error(rds[0].ctx)
            else:
                assert all(rc == piko.PIKO_OK for rc in rcs.values()), rcs
                r0 = rds[0]
                assert np.array_equal(r0.primid().cpu().numpy(), ref["primid"])
                assert np.array_equal(r0.depth.cpu().numpy().view(np.uint32), ref["depth"].view(np.uint32))
    finally:
        for rd in rds[1:] + rds[:1]:
            rd.close()
