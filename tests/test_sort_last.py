"""Sort-last multi-GPU path ("Tiled Depth-Based
Composition", Table 1).

Every rank renders a contiguous triangle range over the whole screen into
packed (depth, primID) keys with GLOBAL primIDs; rank 0 takes the element-wise
minimum (ncclReduce(ncclMin, ncclUint64)) and shades.  The pin is a property of
the method, not of the code: the per-pixel lexicographic minimum over all
triangles equals the minimum over the ranges' minima (min is associative and
commutative), so the composed key image must equal the oracle's full frame.

* CPU: the range plan (host-only library call) partitions [0, T) into
  contiguous, 4-aligned, balanced ranges; a gloo world_size-2 min-reduce of the
  oracle's per-range key images reassembles the full-frame keys.
* GPU (one device, virtual ranks): each rank's key image from the tile kernel
  equals the oracle's image of its range (+ range base), and the resolve of
  their element-wise minimum equals the oracle frame bit for bit.
"""
from __future__ import annotations

import socket

import numpy as np
import pytest

import scenes

CLEAR = np.uint64(0xFFFFFFFFFFFFFFFF)
SIGN = np.uint64(1 << 63)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _range_keys(oracle_lib, s, t0, t1):
    """Oracle key image of triangles [t0, t1) with global primIDs."""
    k = oracle_lib.render(s.verts, s.idx[t0:t1], s.mvp, s.light, s.W, s.H, want_keys=True)["keys"]
    return np.where(k == CLEAR, k, k + np.uint64(t0))


def _untile(tiles, bw, bh, W, H):
    """u64[NB][bw*bh] tile-major key image -> u64[H][W]."""
    binsX, binsY = -(-W // bw), -(-H // bh)
    img = tiles.reshape(binsY, binsX, bh, bw).transpose(0, 2, 1, 3).reshape(binsY * bh, binsX * bw)
    return img[:H, :W]


def test_triangle_ranges_partition():
    import paper_1404_6293_b200 as piko
    for T in (0, 1, 5, 17, 1000, 1_000_003):
        for R in (1, 2, 3, 4, 8):
            rs = [piko.piko_triangle_range(T, r, R) for r in range(R)]
            assert rs[0][0] == 0 and rs[-1][1] == T
            for (a0, a1), (b0, b1) in zip(rs, rs[1:]):
                assert a1 == b0
            for t0, t1 in rs:
                assert t0 % 4 == 0 and t0 <= t1
                assert t1 - t0 <= -(-T // R) + 4
    with pytest.raises(piko.PikoError):
        piko.piko_triangle_range(10, 2, 2)


def _gloo_worker(rank, world, port, img, result):
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    # gloo has no unsigned MIN: flip the sign bit, an order-preserving map of
    # u64 onto i64 (NCCL reduces ncclUint64 directly)
    t = torch.from_numpy((img ^ SIGN).view(np.int64).copy())
    dist.reduce(t, dst=0, op=dist.ReduceOp.MIN)
    if rank == 0:
        result["img"] = t.numpy().view(np.uint64) ^ SIGN
    dist.destroy_process_group()


def test_gloo_min_reduce_reassembles_frame(oracle_lib):
    import multiprocessing as mp
    import paper_1404_6293_b200 as piko
    s = scenes.scene_soup(3000, 160, 96, seed=81, name="soup")
    T = s.idx.shape[0]
    imgs = [_range_keys(oracle_lib, s, *piko.piko_triangle_range(T, r, 2)) for r in range(2)]
    full = oracle_lib.render(s.verts, s.idx, s.mvp, s.light, s.W, s.H, want_keys=True)["keys"]
    assert not np.array_equal(imgs[0], full) and not np.array_equal(imgs[1], full)
    port = _free_port()
    result = {}
    ctx = mp.get_context("spawn")
    p = ctx.Process(target=_gloo_worker, args=(1, 2, port, imgs[1], {}))
    p.start()
    _gloo_worker(0, 2, port, imgs[0], result)
    p.join(timeout=120)
    assert p.exitcode == 0
    assert np.array_equal(result["img"], full)


@pytest.mark.gpu
@pytest.mark.parametrize("name,R", [("c2", 2), ("c2", 3), ("soup", 4)])
def test_gpu_sort_last_virtual_ranks(oracle_lib, name, R):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    import paper_1404_6293_b200 as piko
    s = scenes.scene_c2() if name == "c2" else scenes.scene_soup(20000, 333, 200, seed=82, name="soup")
    bw = 16
    dev = torch.device("cuda:0")
    v = torch.from_numpy(s.verts).to(dev)
    i = torch.from_numpy(s.idx).to(dev)
    T = s.idx.shape[0]
    rds = [piko.Renderer(s.W, s.H, bw, device=dev) for _ in range(R)]
    for r, rd in enumerate(rds):
        piko.piko_set_multi(rd.ctx, piko.PIKO_MULTI_SORT_LAST)
        piko.piko_set_partition(rd.ctx, r, R)
    n = piko.piko_tile_keys_count(rds[0].ctx)
    NB = (-(-s.W // bw)) * (-(-s.H // bw))
    assert n == NB * bw * bw  # every rank owns every bin
    keys = torch.empty((R, n), dtype=torch.int64, device=dev)
    for r, rd in enumerate(rds):
        piko.piko_draw_tile_keys(rd.ctx, v, i, s.mvp, s.light, keys[r])
    torch.cuda.synchronize()
    host = keys.cpu().numpy().view(np.uint64)
    for r in range(R):
        t0, t1 = piko.piko_triangle_range(T, r, R)
        got = _untile(host[r], bw, bw, s.W, s.H)
        assert np.array_equal(got, _range_keys(oracle_lib, s, t0, t1)), f"rank {r} key image"
    reduced = torch.from_numpy(np.minimum.reduce(host, axis=0).view(np.int64).copy()).to(dev)
    r0 = rds[0]
    piko.piko_resolve_keys(r0.ctx, v, i, s.mvp, s.light, 1, reduced, r0.rgba, r0.depth)
    torch.cuda.synchronize()
    ref = oracle_lib.render(s.verts, s.idx, s.mvp, s.light, s.W, s.H)
    assert np.array_equal(r0.primid().cpu().numpy(), ref["primid"])
    assert np.array_equal(r0.depth.cpu().numpy().view(np.uint32), ref["depth"].view(np.uint32))
    assert np.abs(r0.rgba.cpu().numpy() - ref["rgba"]).max() <= 1e-5
    for rd in rds:
        rd.close()
