"""GPU parity of the CUDA path (through the C ABI) against the CPU oracle.

Bar (BASELINE.json north_star): bin lists, coverage, depth and primID
bit-exact; RGB within 1e-5 absolute.  Every input is a seeded synthetic scene
(scenes/), the oracle (oracle/) is independent of the CUDA path.
"""
from __future__ import annotations

import numpy as np
import pytest

import scenes

pytestmark = pytest.mark.gpu

RGB_TOL = 1e-5


@pytest.fixture(scope="module")
def env(oracle_lib):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    import paper_1404_6293_b200 as piko
    return piko, oracle_lib, torch


def gpu_render(env, s, bw, bh=None, cov=True, partition=None, sync=None, indexed=True,
               pipeline=None, frames=1, shader=None):
    piko, _, torch = env
    bh = bw if bh is None else bh
    dev = torch.device("cuda:0")
    verts = torch.from_numpy(np.ascontiguousarray(s.verts)).to(dev)
    idx = torch.from_numpy(np.ascontiguousarray(s.idx)).to(dev)
    r = piko.Renderer(s.W, s.H, bw, bh, device=dev)
    if cov:
        piko.piko_set_debug(r.ctx, piko.PIKO_DEBUG_COVERAGE_COUNT)
    if partition is not None:
        piko.piko_set_partition(r.ctx, *partition)
        r.rgba.fill_(float("nan"))
        r.depth.fill_(float("nan"))
    if sync is not None:
        piko.piko_set_sync(r.ctx, sync)
    if pipeline is not None:
        piko.piko_set_pipeline(r.ctx, pipeline)
    if shader is not None:
        piko.piko_set_shader_cost(r.ctx, *shader)
    for _ in range(frames):
        r.draw(verts, idx, s.mvp, s.light, indexed=indexed)
    torch.cuda.synchronize()
    out = {"rgba": r.rgba.cpu().numpy(), "depth": r.depth.cpu().numpy(),
           "primid": r.primid().cpu().numpy()}
    if cov:
        out["covcount"] = r.coverage().cpu().numpy().view(np.uint32)
    if pipeline in (None, piko.PIKO_PIPE_BINNED):
        st, pr = r.bins()
        out["bin_start"], out["bin_prims"] = st.cpu().numpy(), pr.cpu().numpy()
    out["stats"] = r.stats()
    r.close()
    return out


def assert_frame_equal(got, ref, cov=True):
    assert np.array_equal(got["primid"], ref["primid"]), \
        f"primID mismatch at {np.argwhere(got['primid'] != ref['primid'])[:5].tolist()}"
    gd, rd = got["depth"].view(np.uint32), ref["depth"].view(np.uint32)
    assert np.array_equal(gd, rd), f"depth mismatch at {np.argwhere(gd != rd)[:5].tolist()}"
    if cov:
        assert np.array_equal(got["covcount"], ref["covcount"]), "coverage mismatch"
    err = np.abs(got["rgba"] - ref["rgba"]).max()
    assert err <= RGB_TOL, err


def assert_bins_equal(got, env, s, bw, bh=None, rank=0, nranks=1):
    bh = bw if bh is None else bh
    start, prims = env[1].bins(s.verts, s.idx, s.mvp, s.W, s.H, bw, bh, rank, nranks)
    assert np.array_equal(got["bin_start"], start), "bin_start mismatch"
    assert np.array_equal(got["bin_prims"], prims), "bin_prims mismatch"


def oracle_frame(env, s, cov=True):
    return env[1].render(s.verts, s.idx, s.mvp, s.light, s.W, s.H, want_covcount=cov)


@pytest.fixture(params=["fused", "separate"])
def vs(request, monkeypatch):
    """Vertex-stage mode of the contexts created in the test: transform fused
    into k_setup or the separate k_vertex stage, forced through
    PIKO_SEPARATE_VS (read by piko_create; unset = chosen per frame from V/T)."""
    monkeypatch.setenv("PIKO_SEPARATE_VS", "1" if request.param == "separate" else "0")
    return request.param


# ------------------------------------------------------------------------------
@pytest.mark.parametrize("bw,bh", [(8, 8), (16, 16), (32, 32), (64, 64), (8, 32), (64, 16)])
def test_c1_all_bin_sizes(env, bw, bh):
    s = scenes.scene_c1()
    got = gpu_render(env, s, bw, bh)
    assert_frame_equal(got, oracle_frame(env, s))
    assert_bins_equal(got, env, s, bw, bh)


@pytest.mark.parametrize("bw", [8, 16, 32, 64])
def test_soup_ragged_screen(env, bw):
    """Random soup on a 200x120 screen (partial edge bins in x and y), incl.
    triangles straddling the screen edge and the guard band."""
    s = scenes.scene_soup(20000, 200, 120, seed=21, name="soup", bin_sizes=(bw,))
    got = gpu_render(env, s, bw)
    assert_frame_equal(got, oracle_frame(env, s))
    assert_bins_equal(got, env, s, bw)


def test_large_triangles_int64_path(env):
    """Triangles far larger than 128 px (int64 edge path), some covering the
    whole screen, mixed with tiny ones; perspective camera."""
    rng = np.random.default_rng(31)
    W, H = 640, 480
    T = 400
    big = rng.uniform(-3, 3, (T, 3, 3))
    big[:, :, 2] = rng.uniform(-20, -1.5, (T, 3))
    small = big.mean(1, keepdims=True) + 0.01 * rng.normal(size=(T, 3, 3))
    pos = np.concatenate([big, small], 0).reshape(-1, 3).astype(np.float32)
    verts = scenes.pack_verts(pos, scenes.random_unit(rng, pos.shape[0]))
    idx = np.arange(pos.shape[0], dtype=np.int32).reshape(-1, 3)
    s = scenes.Scene("big", W, H, (16,), verts, idx, scenes.perspective_mvp())
    for bw in (8, 16, 64):
        got = gpu_render(env, s, bw)
        assert_frame_equal(got, oracle_frame(env, s))
        assert_bins_equal(got, env, s, bw)


def test_capacity_overflow_regrows(env):
    """Few full-screen triangles -> P far above the initial pair capacity: the
    checked draw regrows and re-issues, the frame is still exact."""
    tris = [[(-10.0, -10.0), (3000.0, -10.0), (-10.0, 3000.0)]] * 6 + \
           [[(1024.0, 768.0), (-1000.0, 768.0), (1024.0, -1000.0)]] * 6
    from tests.helpers import pixel_scene
    zs = np.linspace(0.1, 0.9, 12)[:, None].repeat(3, 1)
    v, i, m = pixel_scene(tris, zs, 1024, 768)
    s = scenes.Scene("cap", 1024, 768, (8,), v, i, m)
    got = gpu_render(env, s, 8)
    assert got["stats"]["n_pairs"] == 12 * 128 * 96
    assert_frame_equal(got, oracle_frame(env, s))
    assert_bins_equal(got, env, s, 8)


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_north_star_piko_draw_without_vertex_count(env, name, vs):
    """piko_draw (no n_verts; derived on device as max(idx)+1) == oracle."""
    s = scenes.make(name)
    got = gpu_render(env, s, 16, indexed=False)
    assert_frame_equal(got, oracle_frame(env, s))
    assert_bins_equal(got, env, s, 16)


def test_sparse_indices_vertex_overflow_regrows(env, vs):
    """piko_draw with indices far beyond 3*n_tris: the vertex-stage capacity
    overflows, grows and the frame is re-issued; still exact."""
    s = scenes.scene_soup(50, 128, 96, seed=61, name="sparse")
    V = 200000
    verts = np.zeros((V, 8), np.float32)
    rng = np.random.default_rng(62)
    far = rng.choice(np.arange(1000, V), size=s.verts.shape[0], replace=False)
    verts[far] = s.verts
    sp = scenes.Scene("sparse", s.W, s.H, (16,), verts, far[s.idx].astype(np.int32), s.mvp)
    got = gpu_render(env, sp, 16, indexed=False)
    assert_frame_equal(got, oracle_frame(env, sp))
    assert_bins_equal(got, env, sp, 16)
    fp = gpu_render(env, sp, 16, indexed=False, pipeline=env[0].PIKO_PIPE_FREEPIPE)
    assert_frame_equal(fp, oracle_frame(env, sp))


def test_empty_and_all_culled(env):
    piko, _, torch = env
    s = scenes.scene_c1()
    e = scenes.Scene("empty", 64, 64, (8,), s.verts, s.idx[:0], s.mvp)
    got = gpu_render(env, e, 8)
    assert (got["primid"] == -1).all() and (got["depth"] == 1.0).all() and (got["rgba"] == 0).all()
    assert got["stats"]["n_pairs"] == 0 and (got["bin_start"] == 0).all()
    # everything behind the camera
    c = scenes.Scene("culled", 64, 64, (8,), s.verts, s.idx, scenes.perspective_mvp(aspect=1.0))
    got = gpu_render(env, c, 8)
    assert_frame_equal(got, oracle_frame(env, c))


def test_c2_full(env, vs):
    s = scenes.scene_c2()
    got = gpu_render(env, s, 16)
    assert_frame_equal(got, oracle_frame(env, s))
    assert_bins_equal(got, env, s, 16)


@pytest.mark.parametrize("bw", [8, 16, 32, 64])
def test_c3_full_bin_sweep(env, bw):
    s = scenes.scene_c3()
    got = gpu_render(env, s, bw)
    assert_frame_equal(got, oracle_frame(env, s))
    assert_bins_equal(got, env, s, bw)


def test_c4_full(env):
    s = scenes.scene_c4()
    got = gpu_render(env, s, 16, cov=False)
    assert_frame_equal(got, oracle_frame(env, s, cov=False), cov=False)
    assert_bins_equal(got, env, s, 16)


@pytest.mark.parametrize("bw", [16, 8])
def test_c5_full_planar_partition(env, bw):
    s = scenes.scene_c5()
    got = gpu_render(env, s, bw)
    # planar partition: every pixel covered exactly once (property at full size)
    assert got["covcount"].min() == 1 and got["covcount"].max() == 1
    assert_frame_equal(got, oracle_frame(env, s))
    assert_bins_equal(got, env, s, bw)


def test_determinism_byte_identical(env):
    s = scenes.scene_soup(50000, 320, 240, seed=41, name="soup")
    a = gpu_render(env, s, 16)
    b = gpu_render(env, s, 16)
    for k in ("rgba", "depth", "primid", "covcount", "bin_start", "bin_prims"):
        assert a[k].tobytes() == b[k].tobytes(), k


@pytest.mark.parametrize("bw", [8, 32])
def test_many_frames_same_context(env, bw):
    """Races show up as frame-to-frame differences: 12 back-to-back frames in
    one context (async mode, no host sync between them) are all exact."""
    piko, _, torch = env
    s = scenes.scene_c3()
    ref = oracle_frame(env, s, cov=False)
    ostart, oprims = env[1].bins(s.verts, s.idx, s.mvp, s.W, s.H, bw, bw)
    dev = torch.device("cuda:0")
    verts = torch.from_numpy(s.verts).to(dev)
    idx = torch.from_numpy(s.idx).to(dev)
    r = piko.Renderer(s.W, s.H, bw, device=dev)
    r.draw(verts, idx, s.mvp, s.light)            # checked: capacity settles
    piko.piko_set_sync(r.ctx, piko.PIKO_SYNC_ASYNC)
    outs = []
    for k in range(12):
        r.draw(verts, idx, s.mvp, s.light)
        outs.append((r.rgba.clone(), r.depth.clone(), r.primid()))
    assert piko.piko_finish(r.ctx) == piko.PIKO_OK
    st, pr = r.bins()
    assert np.array_equal(st.cpu().numpy(), ostart) and np.array_equal(pr.cpu().numpy(), oprims)
    for rgba, depth, prim in outs:
        got = {"rgba": rgba.cpu().numpy(), "depth": depth.cpu().numpy(), "primid": prim.cpu().numpy()}
        assert_frame_equal(got, ref, cov=False)
    r.close()


@pytest.mark.parametrize("R", [2, 3, 4])
def test_virtual_rank_partition(env, R):
    """Sort-first partition on one GPU: rank r writes exactly its bins
    (b mod R == r); the union over ranks is the full frame; per-rank bin lists
    equal the oracle's rank-filtered lists."""
    s = scenes.scene_soup(30000, 256, 200, seed=51, name="soup")
    full = oracle_frame(env, s)
    bw = 16
    binsX = -(-s.W // bw)
    ys, xs = np.mgrid[0:s.H, 0:s.W]
    owner = ((ys // bw) * binsX + xs // bw) % R
    merged = {k: np.zeros_like(full[k]) for k in ("rgba", "depth", "primid", "covcount")}
    for r in range(R):
        got = gpu_render(env, s, bw, partition=(r, R))
        mine = owner == r
        assert np.isnan(got["depth"][~mine]).all(), "rank wrote pixels it does not own"
        for k in merged:
            merged[k][mine] = got[k][mine]
        assert_bins_equal(got, env, s, bw, rank=r, nranks=R)
    assert_frame_equal(merged, full)


def test_async_mode_and_finish(env):
    piko, _, torch = env
    s = scenes.scene_c2()
    got = gpu_render(env, s, 16, sync=piko.PIKO_SYNC_ASYNC)
    assert_frame_equal(got, oracle_frame(env, s))


def test_draw_host_e2e_matches_device_path(env):
    piko, _, torch = env
    s = scenes.scene_c2()
    r = piko.Renderer(s.W, s.H, 16)
    hv = torch.from_numpy(s.verts).pin_memory()
    hi = torch.from_numpy(s.idx).pin_memory()
    rgba = torch.empty((s.H, s.W, 4), dtype=torch.float32).pin_memory()
    depth = torch.empty((s.H, s.W), dtype=torch.float32).pin_memory()
    piko.piko_draw_host(r.ctx, hv, hi, s.mvp, s.light, rgba, depth)
    ref = oracle_frame(env, s, cov=False)
    assert np.array_equal(depth.numpy().view(np.uint32), ref["depth"].view(np.uint32))
    assert np.abs(rgba.numpy() - ref["rgba"]).max() <= RGB_TOL
    r.close()


def test_draw_host_async_pipelined_frames(env):
    """piko_draw_host_async: six frames of two alternating views (so a slot or
    stream mix-up shows) enqueued back to back into six pinned host buffers,
    then one synchronisation -- every frame bit-exact vs the oracle (c2 first
    draws once synchronously so the pair capacity is settled)."""
    piko, _, torch = env
    s = scenes.scene_c2()
    views = [s.mvp, (np.asarray(s.mvp, np.float32).reshape(4, 4) @ np.diag([1.0, 1.0, 1.0, 1.0]).astype(np.float32)
                     @ np.array([[1, 0, 0, 0.3], [0, 1, 0, 0], [0, 0, 1, 0], [0, 0, 0, 1]], np.float32)).reshape(-1)]
    r = piko.Renderer(s.W, s.H, 16)
    hv = torch.from_numpy(s.verts).pin_memory()
    hi = torch.from_numpy(s.idx).pin_memory()
    rgba0 = torch.empty((s.H, s.W, 4), dtype=torch.float32).pin_memory()
    depth0 = torch.empty((s.H, s.W), dtype=torch.float32).pin_memory()
    piko.piko_draw_host(r.ctx, hv, hi, s.mvp, s.light, rgba0, depth0)
    outs = [(torch.empty((s.H, s.W, 4), dtype=torch.float32).pin_memory(),
             torch.empty((s.H, s.W), dtype=torch.float32).pin_memory()) for _ in range(6)]
    st = torch.cuda.current_stream()
    for k, (rgba, depth) in enumerate(outs):
        assert piko.piko_draw_host_async(r.ctx, hv, hi, views[k % 2], s.light, rgba, depth, st) == 0
    st.synchronize()
    assert piko.piko_finish(r.ctx) == 0
    for v in range(2):
        ref = env[1].render(s.verts, s.idx, np.asarray(views[v], np.float32), s.light, s.W, s.H)
        for k in range(v, 6, 2):
            rgba, depth = outs[k]
            assert np.array_equal(depth.numpy().view(np.uint32), ref["depth"].view(np.uint32)), (v, k)
            assert np.abs(rgba.numpy() - ref["rgba"]).max() <= RGB_TOL
    r.close()


def test_argument_validation(env):
    piko, _, torch = env
    s = scenes.scene_c1()
    r = piko.Renderer(64, 64, 8)
    v = torch.from_numpy(s.verts).cuda()
    i = torch.from_numpy(s.idx).cuda()
    assert piko.piko_draw(r.ctx, v, i, -1, s.mvp, s.light, r.rgba, r.depth, check=False) == piko.PIKO_EINVAL
    assert piko.piko_draw(r.ctx, v, i, 16, s.mvp, [0, 0, 0], r.rgba, r.depth, check=False) == piko.PIKO_EINVAL
    assert piko.piko_draw(r.ctx, v, i, 16, s.mvp, [np.nan, 0, 1], r.rgba, r.depth, check=False) == piko.PIKO_EINVAL
    vv = torch.empty(s.verts.size + 1, dtype=torch.float32, device="cuda")[1:].view(-1, 8)
    assert piko.piko_draw(r.ctx, vv, i, 16, s.mvp, s.light, r.rgba, r.depth, check=False) == piko.PIKO_EINVAL
    assert piko.piko_draw(r.ctx, None, None, 16, s.mvp, s.light, r.rgba, r.depth, check=False) == piko.PIKO_EINVAL
    r.close()


# ---- FreePipe design alternative -----------
@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_freepipe_matches_oracle(env, name, vs):
    piko = env[0]
    s = scenes.make(name)
    got = gpu_render(env, s, 16, pipeline=piko.PIKO_PIPE_FREEPIPE, frames=2)
    assert_frame_equal(got, oracle_frame(env, s))


def test_freepipe_ragged_soup_and_piko_draw(env):
    piko = env[0]
    s = scenes.scene_soup(20000, 200, 120, seed=22, name="soup")
    got = gpu_render(env, s, 16, pipeline=piko.PIKO_PIPE_FREEPIPE, indexed=False)
    assert_frame_equal(got, oracle_frame(env, s))


def test_freepipe_and_binned_switch_in_one_context(env):
    """Switching pipelines inside one context keeps both exact (resets the
    binned path's control block)."""
    piko, _, torch = env
    s = scenes.scene_c2()
    ref = oracle_frame(env, s, cov=False)
    dev = torch.device("cuda:0")
    v = torch.from_numpy(s.verts).to(dev)
    i = torch.from_numpy(s.idx).to(dev)
    r = piko.Renderer(s.W, s.H, 16, device=dev)
    for pipe in (0, 1, 0, 1, 0):
        piko.piko_set_pipeline(r.ctx, pipe)
        r.draw(v, i, s.mvp, s.light)
        got = {"rgba": r.rgba.cpu().numpy(), "depth": r.depth.cpu().numpy(),
               "primid": r.primid().cpu().numpy()}
        assert_frame_equal(got, ref, cov=False)
    r.close()


# ---- API behaviour ---------------------------------------------------------------
def test_stats_and_profile(env):
    piko, _, torch = env
    s = scenes.scene_c3()
    dev = torch.device("cuda:0")
    v = torch.from_numpy(s.verts).to(dev)
    i = torch.from_numpy(s.idx).to(dev)
    r = piko.Renderer(s.W, s.H, 16, device=dev)
    piko.piko_set_profiling(r.ctx, 1)
    for _ in range(3):
        r.draw(v, i, s.mvp, s.light)
    prof, n = piko.piko_get_profile(r.ctx)
    assert n == 3 and all(ms >= 0 for ms in prof.values()) and prof["tile"] > 0
    st = r.stats()
    ostart, oprims = env[1].bins(s.verts, s.idx, s.mvp, s.W, s.H, 16, 16)
    assert st["n_pairs"] == len(oprims) and st["n_bins"] == len(ostart) - 1
    oi, _ = env[1].setup(s.verts, s.idx, s.mvp, s.W, s.H)
    assert st["n_live"] == int(oi[:, 0].sum())
    # c3 is a shared-vertex mesh (2V <= 3T): separate vertex stage; count-matrix
    # AssignBin (the default): k_vertex, k_setup, k_cm_scan, k_cm_scatter, k_tile
    assert st["radix_passes"] == 2 and st["kernels_per_frame"] == 5
    assert st["assign_mode"] == 1
    r.close()


def test_async_overflow_is_reported_then_recovers(env):
    """ASYNC mode: a frame that overflows the pair capacity is reported by
    piko_finish (PIKO_ECAPACITY) and the capacity grows; the next frame is exact."""
    piko, _, torch = env
    from tests.helpers import pixel_scene
    tris = [[(-10.0, -10.0), (3000.0, -10.0), (-10.0, 3000.0)]] * 40
    zs = np.linspace(0.1, 0.9, 40)[:, None].repeat(3, 1)
    v, i, m = pixel_scene(tris, zs, 1024, 768)
    s = scenes.Scene("cap", 1024, 768, (8,), v, i, m)
    dev = torch.device("cuda:0")
    vt, it = torch.from_numpy(v).to(dev), torch.from_numpy(i).to(dev)
    r = piko.Renderer(1024, 768, 8, device=dev)
    piko.piko_set_sync(r.ctx, piko.PIKO_SYNC_ASYNC)
    r.draw(vt, it, m, s.light)
    assert piko.piko_finish(r.ctx) == piko.PIKO_ECAPACITY
    r.draw(vt, it, m, s.light)
    assert piko.piko_finish(r.ctx) == piko.PIKO_OK
    ref = oracle_frame(env, s, cov=False)
    got = {"rgba": r.rgba.cpu().numpy(), "depth": r.depth.cpu().numpy(), "primid": r.primid().cpu().numpy()}
    assert_frame_equal(got, ref, cov=False)
    r.close()


@pytest.mark.parametrize("bw,bh", [(8, 32), (32, 8), (64, 16)])
def test_c3_non_square_bins(env, bw, bh):
    s = scenes.scene_c3()
    got = gpu_render(env, s, bw, bh, cov=False)
    assert_frame_equal(got, oracle_frame(env, s, cov=False), cov=False)
    assert_bins_equal(got, env, s, bw, bh)


@pytest.mark.parametrize("W,H", [(16384, 24), (24, 16384), (1, 1), (4097, 3)])
def test_extreme_screens(env, W, H):
    """Maximum width / height (guard band limit R2), 1x1 and odd sizes."""
    s = scenes.scene_soup(3000, W, H, seed=81, name="soup")
    got = gpu_render(env, s, 16, cov=False)
    assert_frame_equal(got, oracle_frame(env, s, cov=False), cov=False)
    assert_bins_equal(got, env, s, 16)


@pytest.mark.parametrize("T", [200, 1000, 3000])
def test_large_triangle_queue_spill_and_fallback(env, T):
    """One 64x64 bin (single-bin grid: the work item is the whole pair list)
    with T medium triangles (clipped area > TINY_AREA): T=200 fits the shared
    queue (256), 1000 spills to the global overflow region (1024 per CTA), 3000
    also takes the warp-cooperative fallback.  Bit-exact either way."""
    s = scenes.scene_soup(T, 64, 64, seed=95 + T, name="spill")
    got = gpu_render(env, s, 64)
    assert_frame_equal(got, oracle_frame(env, s))
    assert_bins_equal(got, env, s, 64)


# ------------------------------------------------------------------------------
# Pixel-shader complexity knob (NEXT-3): extra per-fragment
# (forward) or per-pixel (deferred) work must leave every output bit unchanged.
@pytest.mark.parametrize("pipeline", ["binned", "freepipe", "baseline"])
@pytest.mark.parametrize("iters,forward", [(64, 1), (64, 0), (1000, 1)])
def test_shader_cost_output_invariant(env, pipeline, iters, forward):
    piko = env[0]
    pl = {"binned": piko.PIKO_PIPE_BINNED, "freepipe": piko.PIKO_PIPE_FREEPIPE,
          "baseline": piko.PIKO_PIPE_BASELINE}[pipeline]
    for s, bw in ((scenes.scene_c1(), 8),
                  (scenes.scene_soup(20000, 200, 120, seed=23, name="soup", bin_sizes=(16,)), 16)):
        got = gpu_render(env, s, bw, pipeline=pl, shader=(iters, forward), frames=2)
        assert_frame_equal(got, oracle_frame(env, s))
        if pipeline == "binned":
            assert_bins_equal(got, env, s, bw)


def test_shader_cost_rejects_bad_args(env):
    piko = env[0]
    r = piko.Renderer(64, 64, 8)
    for args in ((-1, 0), (piko.PIKO_MAX_SHADER_ITERS + 1, 1), (4, 2)):
        with pytest.raises(piko.PikoError):
            piko.piko_set_shader_cost(r.ctx, *args)
    piko.piko_set_shader_cost(r.ctx, 0, 0)
    r.close()


# ------------------------------------------------------------------------------
# Baseline design alternative (NEXT-3): one kernel per stage with
# fragment buffers in HBM -- the same frame, bit for bit.
@pytest.mark.parametrize("indexed", [True, False])
def test_baseline_pipeline(env, indexed):
    piko = env[0]
    for s, bw in ((scenes.scene_c1(), 8),
                  (scenes.scene_soup(20000, 200, 120, seed=29, name="soup", bin_sizes=(16,)), 16),
                  (scenes.scene_c2(), 16)):
        got = gpu_render(env, s, bw, pipeline=piko.PIKO_PIPE_BASELINE, indexed=indexed, frames=2)
        assert_frame_equal(got, oracle_frame(env, s))


def test_baseline_fragment_overflow_regrows(env):
    """Depth complexity 64 on 64x64 (131072 fragments against an initial
    capacity of 4 W H = 16384): the checked draw grows the fragment buffers
    and re-issues; the frame matches the oracle."""
    from tests.helpers import pixel_scene
    piko = env[0]
    rng = np.random.default_rng(31)
    tris, zw = [], []
    for k in range(64):
        tris.append([(-8.0, -8.0), (140.0, -8.0), (-8.0, 140.0)] if k % 2 else
                    [(72.0, 72.0), (-76.0, 72.0), (72.0, -76.0)])
        zw.append(float(rng.uniform(0.1, 0.9)))
    verts, idx, mvp = pixel_scene(tris, zw, 64, 64)
    s = scenes.Scene("stack", 64, 64, (8,), verts, idx, mvp)
    got = gpu_render(env, s, 8, pipeline=piko.PIKO_PIPE_BASELINE)
    assert got["stats"]["n_pairs"] == 64 * 64 * 64  # both triangles cover every pixel centre
    assert_frame_equal(got, oracle_frame(env, s))


# ---- round 2: the exact benchmarked instantiation and the oracle-pin scenes --
ASSIGN_ENV = {"chunk-list": {"PIKO_CL": "1"}, "count-matrix": {"PIKO_CL": "0", "PIKO_CM": "1"},
              "radix": {"PIKO_CL": "0", "PIKO_CM": "0"}}
ASSIGN_MODE = {"chunk-list": 2, "count-matrix": 1, "radix": 0}


@pytest.mark.parametrize("assign", ["chunk-list", "count-matrix", "radix"])
def test_c3_b16_cov_off_bench_variant(env, assign, monkeypatch):
    """The instantiation bench.py times: c3, 16x16 bins, coverage counting off
    (k_tile<16,16,256,COV=0,KEYS=0>), the separate vertex stage (c3 shares
    vertices: chosen automatically), AssignBin as configured (count matrix by
    default; the chunk lists and the radix passes forced) -- bit-exact vs the
    oracle."""
    for k, v in ASSIGN_ENV[assign].items():
        monkeypatch.setenv(k, v)
    monkeypatch.delenv("PIKO_SEPARATE_VS", raising=False)
    s = scenes.scene_c3()
    got = gpu_render(env, s, 16, cov=False, frames=3)
    assert_frame_equal(got, oracle_frame(env, s, cov=False), cov=False)
    assert_bins_equal(got, env, s, 16)
    assert got["stats"]["assign_mode"] == ASSIGN_MODE[assign]
    assert got["stats"]["kernels_per_frame"] == (4 if assign == "chunk-list" else 5)


@pytest.mark.parametrize("assign", ["chunk-list", "count-matrix", "radix"])
@pytest.mark.parametrize("cfg,bw", [("c2", 16), ("c2", 8), ("c1", 8)])
def test_assign_modes_agree(env, assign, cfg, bw, monkeypatch):
    """Every AssignBin mode gives the oracle's bin lists and frame (c2: many
    chunks, 2.2 pairs per triangle; 8-px bins: NB = 12288 > CL_MAX_NB, so the
    chunk-list request falls through to the count matrix)."""
    for k, v in ASSIGN_ENV[assign].items():
        monkeypatch.setenv(k, v)
    s = scenes.make(cfg)
    got = gpu_render(env, s, bw, frames=2)
    assert_frame_equal(got, oracle_frame(env, s))
    assert_bins_equal(got, env, s, bw)
    NB = ((s.W + bw - 1) // bw) * ((s.H + bw - 1) // bw)
    want = ASSIGN_MODE[assign] if not (assign == "chunk-list" and NB > 4096) else 1
    assert got["stats"]["assign_mode"] == want


def test_chunk_list_overflow_falls_back(env, monkeypatch):
    """A bin that collects more than CLB_GRP = 2048 groups of 32 triangles
    (3000 scattered one-bin triangles x 32 stride: one per group, all in bin 0,
    plus fill): the frame reports the overflow, the context switches to the
    count matrix, and the checked draw re-issues it -- frame and bin lists exact."""
    from tests.helpers import pixel_scene
    tris = []
    for k in range(2100 * 32):
        if k % 32 == 0:
            tris.append([(1.5, 1.5), (5.5, 1.5), (1.5, 5.5)])  # bin 0 (8-px bins)
        else:
            tris.append([(300.5, 300.5), (300.5, 300.5), (300.5, 300.5)])  # degenerate: culled
    verts, idx, mvp = pixel_scene(tris, 0.5, 512, 512)
    s = scenes.Scene("cl_overflow", 512, 512, (8,), verts, idx, mvp)
    monkeypatch.setenv("PIKO_CL", "1")
    got = gpu_render(env, s, 8, frames=2)
    assert got["stats"]["n_pairs"] == 2100
    assert got["stats"]["assign_mode"] == 1
    assert_frame_equal(got, oracle_frame(env, s))
    assert_bins_equal(got, env, s, 8)


def _pin_scenes():
    """The scenes of the round-2 oracle pins (tests/test_oracle_pins.py):
    snap ties, guard band, near epsilon, zero area with a non-empty rect,
    zero depth at the range boundary."""
    from tests.helpers import pixel_scene
    W = H = 64
    out = []
    tris, zw = [], []
    for x in (10 + 1 / 512, 11 + 3 / 512, -1 / 512):
        tris.append([(x, 0.5), (x + 20.0, 0.5), (x, 20.5)])
    for x in (16383.75, 16384.0, 16384.5):
        tris.append([(0.5, 0.5), (x, 0.5), (0.5, 16.5)])
    tris.append([(-16384.5, 0.5), (40.5, 0.5), (40.5, 16.5)])
    tris += [[(0.5, 0.5), (5.5, 0.5), (10.5, 0.5)], [(0.5, 0.5), (10.5, 0.5), (10.5, 0.5)]]
    zw = [[0.5] * 3] * len(tris)
    tris += [[(0.5, 0.5), (40.5, 0.5), (0.5, 40.5)], [(0.5, 0.5), (32.5, 0.5), (0.5, 32.5)]]
    zw += [[2.0 ** -25] * 3, [-0.125, 0.375, -0.125]]
    v, i, m = pixel_scene(tris, np.array(zw), W, H)
    out.append(scenes.Scene("pins", W, H, (8,), v, i, m))
    for w0 in (2e-6, 1.0000001e-6, 5e-7):
        M = np.zeros(16, np.float32)
        M[0] = M[5] = 1.0
        M[15] = np.float32(w0)
        ndc = np.array([[-0.5, -0.5], [0.5, -0.5], [0.0, 0.5]])
        pos = np.concatenate([ndc * np.float32(w0), np.zeros((3, 1))], 1).astype(np.float32)
        verts = scenes.pack_verts(pos, np.tile([0, 0, 1.0], (3, 1)).astype(np.float32))
        out.append(scenes.Scene(f"weps{w0}", W, H, (8,), verts, np.arange(3, dtype=np.int32).reshape(1, 3), M))
    return out


@pytest.mark.parametrize("k", range(4))
def test_oracle_pin_scenes_match(env, k, vs):
    s = _pin_scenes()[k]
    got = gpu_render(env, s, 8)
    assert_frame_equal(got, oracle_frame(env, s))
    assert_bins_equal(got, env, s, 8)


def test_piko_draw_is_asynchronous(env):
    """piko_draw returns once the frame is enqueued.  The stream
    is held by a long device sleep; 8 c3 frames through the north-star
    piko_draw (C default: async) all return while the first frame's end event
    is still pending (cudaEventQuery), then piko_finish reports OK and the
    last frame is exact."""
    piko, _, torch = env
    s = scenes.scene_c3()
    dev = torch.device("cuda:0")
    v, i = torch.from_numpy(s.verts).to(dev), torch.from_numpy(s.idx).to(dev)
    r = piko.Renderer(s.W, s.H, 16, device=dev, sync="async")
    r.draw(v, i, s.mvp, s.light, indexed=False)  # warm-up (allocations)
    assert piko.piko_finish(r.ctx) == piko.PIKO_OK
    st = torch.cuda.current_stream()
    torch.cuda._sleep(2_000_000_000)  # ~1 s of device time ahead of the frames
    ev = torch.cuda.Event()
    for k in range(8):
        assert r.draw(v, i, s.mvp, s.light, indexed=False) == piko.PIKO_OK
        if k == 0:
            ev.record(st)
    assert not ev.query(), "a piko_draw call waited for the device"
    assert piko.piko_finish(r.ctx) == piko.PIKO_OK
    assert ev.query()
    ref = oracle_frame(env, s, cov=False)
    got = {"rgba": r.rgba.cpu().numpy(), "depth": r.depth.cpu().numpy(), "primid": r.primid().cpu().numpy()}
    assert_frame_equal(got, ref, cov=False)
    r.close()


def test_async_overflow_reported_by_next_draw(env):
    """an async frame that overflows is reported (once) by the next
    piko_draw, which was enqueued with the grown capacity; that frame is exact."""
    piko, _, torch = env
    from tests.helpers import pixel_scene
    tris = [[(-10.0, -10.0), (3000.0, -10.0), (-10.0, 3000.0)]] * 40
    zs = np.linspace(0.1, 0.9, 40)[:, None].repeat(3, 1)
    v, i, m = pixel_scene(tris, zs, 1024, 768)
    s = scenes.Scene("cap", 1024, 768, (8,), v, i, m)
    dev = torch.device("cuda:0")
    vt, it = torch.from_numpy(v).to(dev), torch.from_numpy(i).to(dev)
    r = piko.Renderer(1024, 768, 8, device=dev, sync="async")
    assert r.draw(vt, it, m, s.light, check=False) == piko.PIKO_OK  # enqueued (overflows)
    torch.cuda.synchronize()
    assert r.draw(vt, it, m, s.light, check=False) == piko.PIKO_ECAPACITY  # frame 1's status
    assert piko.piko_finish(r.ctx) == piko.PIKO_OK
    ref = oracle_frame(env, s, cov=False)
    got = {"rgba": r.rgba.cpu().numpy(), "depth": r.depth.cpu().numpy(), "primid": r.primid().cpu().numpy()}
    assert_frame_equal(got, ref, cov=False)
    r.close()


@pytest.mark.parametrize("deferred", ["1", "0"])
@pytest.mark.parametrize("cfg,bw", [("c1", 8), ("c2", 16), ("c3", 16), ("c2", 32)])
def test_deferred_resolve_matches_oracle(env, cfg, bw, deferred, monkeypatch):
    """Keys-only k_tile (empty bins skipped) + the one-pixel-per-thread deferred
    resolve k_shade1 (background of empty bins from the CSR, lean O2 orientation
    from the snapped corners) against the oracle, and the immediate write-back
    beside it."""
    monkeypatch.setenv("PIKO_DEFERRED", deferred)
    s = scenes.make(cfg)
    got = gpu_render(env, s, bw, cov=False, frames=2)
    assert_frame_equal(got, oracle_frame(env, s, cov=False), cov=False)
    assert_bins_equal(got, env, s, bw)


def test_deferred_overflow_frame_is_background_then_exact(env, monkeypatch):
    """An overflowing deferred frame (pair capacity) is reported and re-issued;
    the final frame is exact."""
    monkeypatch.setenv("PIKO_DEFERRED", "1")
    s = scenes.scene_c2()
    got = gpu_render(env, s, 8, cov=False, frames=1)  # 8-px bins: P = 418504 > the initial capacity
    assert_frame_equal(got, oracle_frame(env, s, cov=False), cov=False)


def test_dense_count_matrix_switches_to_radix(env, monkeypatch):
    """Auto AssignBin: an unordered soup's count-matrix rows are dense (most of
    a scatter window's pairs in distinct bins), so after the first frame the
    context ranks frames of that size with the radix passes -- both frames
    exact, the bin lists too; a coherent mesh (c3) stays on the count matrix."""
    monkeypatch.delenv("PIKO_CM", raising=False)
    s = scenes.scene_soup(200000, 960, 540, seed=77, name="soup", bin_sizes=(16,))
    got = gpu_render(env, s, 16, cov=False, frames=2)
    assert got["stats"]["assign_mode"] == 0
    assert_frame_equal(got, oracle_frame(env, s, cov=False), cov=False)
    assert_bins_equal(got, env, s, 16)
