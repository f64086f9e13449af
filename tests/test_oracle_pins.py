"""Pins of the CPU oracle against what the paper and mathematics fix (-m "not gpu").

Each test cites the passage it pins.  None re-types the oracle's formulas: the
checks are hand-computed values (tests/golden/, cited), closed forms, exact
rational re-definitions, invariants (watertightness, order independence) and
library routines (numpy stable argsort, float64 geometry).
"""
from __future__ import annotations

import math

import numpy as np
import pytest

import scenes
from tests.helpers import covered_exact, lattice, load_golden, pixel_scene

L111 = np.array([1.0, 1.0, 1.0], np.float32)


def cross2(a, b):
    return a[0] * b[1] - a[1] * b[0]


def render(oracle_lib, verts, idx, mvp, W, H, light=L111):
    return oracle_lib.render(verts, idx, mvp, light, W, H, want_covcount=True, want_keys=True)


# ---------------------------------------------------------------- coverage ---
def test_right_triangle_six_fragments(oracle_lib):
    """SPEC.md:509 example: (0,0),(4,0),(0,4) -> exactly 6 pixels (golden)."""
    gold = {tuple(int(v) for v in r) for r in load_golden("right_triangle_coverage.txt")}
    for wind in ([(0, 0), (4, 0), (0, 4)], [(0, 0), (0, 4), (4, 0)]):
        v, i, m = pixel_scene([wind], 0.5, 16, 16)
        r = render(oracle_lib, v, i, m, 16, 16)
        got = {(x, y) for y, x in zip(*np.nonzero(r["covcount"]))}
        assert got == gold
        assert r["covcount"].max() == 1


def test_complement_tiles_square_exactly_once(oracle_lib):
    """Top-left rule (R1): (0,0),(4,0),(0,4) + (4,0),(0,4),(4,4)
    cover the 4x4 square exactly once, and nothing else (6 + 10 pixels)."""
    v, i, m = pixel_scene([[(0, 0), (4, 0), (0, 4)], [(4, 0), (4, 4), (0, 4)]], 0.5, 16, 16)
    r = render(oracle_lib, v, i, m, 16, 16)
    cov = r["covcount"]
    assert cov[:4, :4].min() == 1 and cov[:4, :4].max() == 1
    assert cov.sum() == 16
    assert (r["primid"][:4, :4] == 1).sum() == 10


def test_fan_on_pixel_centre_covered_once(oracle_lib):
    """A 7-triangle fan whose shared vertex is exactly the pixel centre
    (8.5, 8.5) covers it once (SURVEY 8(c) pin for O2/O3)."""
    c = (8.5, 8.5)
    ring = [(8.5 + 4 * math.cos(a), 8.5 + 4 * math.sin(a)) for a in np.arange(7) * 2 * math.pi / 7]
    ring = [(round(x * 2) / 2, round(y * 2) / 2) for x, y in ring]
    tris = [[c, ring[k], ring[(k + 1) % 7]] for k in range(7)]
    v, i, m = pixel_scene(tris, 0.5, 16, 16)
    r = render(oracle_lib, v, i, m, 16, 16)
    assert r["covcount"][8, 8] == 1
    assert r["covcount"].max() == 1


@pytest.mark.parametrize("step", [0.5, 1.0 / 256])
def test_coverage_equals_exact_rational_definition(oracle_lib, step):
    """Brute force over every pixel of a 16x16 image: oracle coverage (bbox loop,
    integer edge functions, top-left rule) == the perturbed-sample-point
    definition in exact rationals, for 120 random triangles per lattice,
    including vertices outside the screen and degenerate ones."""
    rng = np.random.default_rng(7 if step == 0.5 else 8)
    W = H = 16
    for _ in range(120):
        xy = np.stack([lattice(rng, 3, -6, 22, step), lattice(rng, 3, -6, 22, step)], 1)
        if rng.random() < 0.05:
            xy[2] = xy[0] + (xy[1] - xy[0]) * 0.5  # collinear -> culled
        v, i, m = pixel_scene([xy], 0.5, W, H)
        cov = render(oracle_lib, v, i, m, W, H)["covcount"]
        want = np.array([[covered_exact(xy, x, y) for x in range(W)] for y in range(H)])
        assert np.array_equal(cov.astype(bool), want), xy
        assert cov.max() <= 1


def test_watertight_jittered_grid(oracle_lib):
    """Planar partition (jittered grid mesh over the whole NDC square, shared
    vertices): every pixel centre is covered exactly once (watertightness)."""
    s = scenes.scene_grid(24, 16, 64, 48, seed=11, name="grid", bin_sizes=(8,))
    r = render(oracle_lib, s.verts, s.idx, s.mvp, s.W, s.H)
    assert r["covcount"].min() == 1 and r["covcount"].max() == 1


def test_shared_edge_pairs_watertight(oracle_lib):
    """adjacent triangles sharing an edge cover each edge pixel
    exactly once -- 1000 random pairs forming a convex quad on the 1/256 lattice:
    coverage count <= 1 everywhere, and == 1 at every centre strictly inside."""
    rng = np.random.default_rng(12)
    W = H = 32
    xs, ys = np.meshgrid(np.arange(W) + 0.5, np.arange(H) + 0.5)
    n_checked = 0
    for _ in range(1000):
        p = np.stack([lattice(rng, 4, 0, 32, 1 / 256), lattice(rng, 4, 0, 32, 1 / 256)], 1)
        # keep only strictly convex quads a, c, b, d (shared diagonal a-b)
        hull = p[[0, 2, 1, 3]]
        cr = [cross2(hull[(k + 1) % 4] - hull[k], hull[(k + 2) % 4] - hull[(k + 1) % 4]) for k in range(4)]
        if not (all(c > 1e-3 for c in cr) or all(c < -1e-3 for c in cr)):
            continue
        a, b, c, d = p
        v, i, m = pixel_scene([[a, b, c], [b, a, d]], 0.5, W, H)
        cov = render(oracle_lib, v, i, m, W, H)["covcount"]
        assert cov.max() <= 1
        # float64 distance from each centre to the quad boundary (signed, inside > 0)
        sgn = 1.0 if cr[0] > 0 else -1.0
        dist = np.full(xs.shape, np.inf)
        for k in range(4):
            e0, e1 = hull[k], hull[(k + 1) % 4]
            nrm = np.array([-(e1 - e0)[1], (e1 - e0)[0]]) * sgn / np.linalg.norm(e1 - e0)
            dist = np.minimum(dist, (xs - e0[0]) * nrm[0] + (ys - e0[1]) * nrm[1])
        inside = dist > 1e-9
        assert (cov[inside] == 1).all()
        n_checked += 1
    assert n_checked > 200


def test_bbox_loop_equals_every_pixel_on_c1(oracle_lib):
    """c1 (16 tris, 64x64): per-triangle coverage from the oracle's bbox loop ==
    the exact rational definition evaluated at every pixel of the image."""
    s = scenes.scene_c1()
    total = np.zeros((64, 64), np.int64)
    for t in range(s.n_tris):
        xy = [(float(s.verts[k, 0]), float(s.verts[k, 1])) for k in s.idx[t]]
        total += np.array([[covered_exact(xy, x, y) for x in range(64)] for y in range(64)])
    r = render(oracle_lib, s.verts, s.idx, s.mvp, 64, 64)
    assert np.array_equal(r["covcount"].astype(np.int64), total)


# --------------------------------------------------------------- transform ---
def test_ortho_viewport_closed_form(oracle_lib):
    """O1 closed form: ortho pixel mvp at power-of-two size maps (x, y) to
    exactly (256x, 256y) subpixels and object z = 2zw-1 to zw."""
    rng = np.random.default_rng(3)
    xy = lattice(rng, 60, -10, 70, 1 / 256).reshape(-1, 3, 2)[:10]
    v, i, m = pixel_scene(xy, 0.375, 64, 64)
    oi, of = oracle_lib.setup(v, i, m, 64, 64)
    for t in range(10):
        X = oi[t, 1:7].reshape(3, 2)
        # corners may be swapped by orientation normalisation (O2)
        want = np.round(xy[t] * 256).astype(np.int64)
        if oi[t, 11]:
            want = want[[0, 2, 1]]
        assert np.array_equal(X, want)
        assert (of[t, :3] == np.float32(0.375)).all()


def test_perspective_transform_vs_float64(oracle_lib):
    """O1 against a float64 evaluation of clip = M (x,y,z,1), GL viewport
    (y down) and depth map: snapped X, Y within 0.5 + fp32 slack subpixels;
    zw within 1e-6; rw within 1e-6 relative.  Pins row-major M, the y flip
    and the [-1,1] -> [0,1] depth map."""
    rng = np.random.default_rng(4)
    W, H = 1024, 768
    M = scenes.perspective_mvp()
    T = 300
    pos = np.stack([rng.uniform(-2, 2, 3 * T), rng.uniform(-1.5, 1.5, 3 * T),
                    rng.uniform(-20, -2, 3 * T)], 1).astype(np.float32)
    verts = scenes.pack_verts(pos, np.tile([0, 0, 1.0], (3 * T, 1)).astype(np.float32))
    idx = np.arange(3 * T, dtype=np.int32).reshape(T, 3)
    oi, of = oracle_lib.setup(verts, idx, M, W, H)
    M64 = M.astype(np.float64).reshape(4, 4)
    clip = np.concatenate([pos.astype(np.float64), np.ones((3 * T, 1))], 1) @ M64.T
    ndc = clip[:, :3] / clip[:, 3:4]
    X = (ndc[:, 0] * 0.5 + 0.5) * W * 256
    Y = (0.5 - ndc[:, 1] * 0.5) * H * 256
    Z = ndc[:, 2] * 0.5 + 0.5
    checked = 0
    for t in range(T):
        if not oi[t, 0]:
            continue
        order = [0, 2, 1] if oi[t, 11] else [0, 1, 2]
        for k, c in enumerate(order):
            g = 3 * t + c
            assert abs(oi[t, 1 + 2 * k] - X[g]) <= 0.5 + 2e-6 * abs(X[g]) + 0.05
            assert abs(oi[t, 2 + 2 * k] - Y[g]) <= 0.5 + 2e-6 * abs(Y[g]) + 0.05
            assert abs(of[t, k] - Z[g]) <= 1e-6
            assert abs(of[t, 3 + k] - 1.0 / clip[g, 3]) <= 1e-6 / clip[g, 3]
        checked += 1
    assert checked > 100


def test_culls(oracle_lib):
    """O1/O2/O4 culls: behind the eye (w < 0), NaN, w below the near epsilon,
    zero area, and a sliver missing every pixel centre -> no coverage, no bins.
    (The guard band, the epsilon's value and the zero-area cull with a
    non-empty sample rect are isolated in the tests below.)"""
    W = H = 64
    M = scenes.perspective_mvp(aspect=1.0)
    pos = np.array([
        [0, 0, 1], [1, 0, 1], [0, 1, 1],               # behind the camera (w < 0)
        [0, 0, -5], [np.nan, 0, -5], [0, 1, -5],       # NaN
        [0, 0, -1e-9], [1e-3, 0, -1e-9], [0, 1e-3, -1e-9],  # w = 1e-9 <= W_EPS (near plane)
        [0, 0, -5], [1, 0, -5], [2, 0, -5],            # zero area
        [0.0, 0.0, -5], [0.0001, 0.0, -5], [0.0, 0.0001, -5],  # misses all centres
    ], np.float32)
    verts = scenes.pack_verts(pos, np.tile([0, 0, 1.0], (15, 1)).astype(np.float32))
    idx = np.arange(15, dtype=np.int32).reshape(5, 3)
    oi, _ = oracle_lib.setup(verts, idx, M, W, H)
    assert oi[:, 0].tolist() == [0, 0, 0, 0, 0]
    r = render(oracle_lib, verts, idx, M, W, H)
    assert r["covcount"].sum() == 0 and (r["primid"] == -1).all()
    start, prims = oracle_lib.bins(verts, idx, M, W, H, 8, 8)
    assert len(prims) == 0


def _live_and_bins(oracle_lib, verts, idx, mvp, W, H):
    oi, _ = oracle_lib.setup(verts, idx, mvp, W, H)
    _, prims = oracle_lib.bins(verts, idx, mvp, W, H, 8, 8)
    return oi, prims


def test_snap_rounds_half_to_even(oracle_lib):
    """R2 (SURVEY 8(c) ledger row 2: `rint`, ties to even): under the exact
    ortho pixel matrix a corner at x = 10 + 1/512 px is 2560.5 subpixels and
    snaps to 2560 (ties away from zero would give 2561); x = 11 + 3/512 ->
    2817.5 -> 2818; x = -1/512 -> -0.5 -> 0 (not -1)."""
    W = H = 64
    for x, want in ((10 + 1 / 512, 2560), (11 + 3 / 512, 2818), (-1 / 512, 0)):
        v, i, m = pixel_scene([[(x, 0.5), (x + 20.0, 0.5), (x, 20.5)]], 0.5, W, H)
        oi, _ = oracle_lib.setup(v, i, m, W, H)
        assert oi[0, 0] == 1 and oi[0, 1] == want, (x, oi[0])
        # the other corners sit exactly on the lattice
        assert sorted([oi[0, 3], oi[0, 5]]) == sorted([want + 5120, want])


def test_guard_band_cull(oracle_lib):
    """R2/R3 guard band (SURVEY 8(c) ledger rows 2-3: cull outside +-2^22
    subpixels = 16384 px, boundary inclusive).  w is exactly 1 under the
    ortho pixel matrix, so the corner's x is exact: x = 16383.75 and x = 16384
    px are kept (the triangle covers centres near the origin and enters bins);
    x = 16384.5 px (4194432 subpixels) culls the triangle.  A 2^24 band or no
    test at all would keep it."""
    W = H = 64
    for x, live in ((16383.75, 1), (16384.0, 1), (16384.5, 0), (-16384.5, 0)):
        v, i, m = pixel_scene([[(0.5, 0.5), (x, 0.5), (0.5, 16.5)]] if x > 0 else
                              [[(x, 0.5), (40.5, 0.5), (40.5, 16.5)]], 0.5, W, H)
        oi, prims = _live_and_bins(oracle_lib, v, i, m, W, H)
        assert oi[0, 0] == live, (x, oi[0])
        assert (len(prims) > 0) == bool(live)


def test_near_plane_epsilon(oracle_lib):
    """R3 ("w <= epsilon ... culled"; SURVEY 8(c) W_EPS = 1e-6):
    a triangle whose clip w is 2e-6 is kept, one at w = 5e-7 is culled, with
    the same NDC footprint (clip = (x, y, 0, w0): xn = x / w0)."""
    W = H = 64
    for w0, live in ((2e-6, 1), (1.0000001e-6, 1), (5e-7, 0), (1e-7, 0)):
        M = np.zeros(16, np.float32)
        M[0] = 1.0
        M[5] = 1.0
        M[15] = np.float32(w0)
        ndc = np.array([[-0.5, -0.5], [0.5, -0.5], [0.0, 0.5]], np.float64)
        pos = np.concatenate([ndc * np.float32(w0), np.zeros((3, 1))], 1).astype(np.float32)
        verts = scenes.pack_verts(pos, np.tile([0, 0, 1.0], (3, 1)).astype(np.float32))
        idx = np.arange(3, dtype=np.int32).reshape(1, 3)
        oi, prims = _live_and_bins(oracle_lib, verts, idx, M, W, H)
        assert oi[0, 0] == live, (w0, oi[0])
        assert (len(prims) > 0) == bool(live)
        r = render(oracle_lib, verts, idx, M, W, H)
        assert (r["covcount"].sum() > 0) == bool(live)


def test_zero_area_with_nonempty_rect_is_culled(oracle_lib):
    """R7 ("degenerate t emits nothing"): collinear corners on the
    pixel-centre row y = 0.5 have a non-empty sample rect (row 0, x 0..10) but
    area2 == 0, so the triangle is culled: no coverage, no bin entry -- also
    when a corner is repeated."""
    W = H = 64
    for tri in ([(0.5, 0.5), (5.5, 0.5), (10.5, 0.5)], [(0.5, 0.5), (10.5, 0.5), (10.5, 0.5)]):
        v, i, m = pixel_scene([tri], 0.5, W, H)
        oi, prims = _live_and_bins(oracle_lib, v, i, m, W, H)
        assert oi[0, 0] == 0 and len(prims) == 0
        assert render(oracle_lib, v, i, m, W, H)["covcount"].sum() == 0


def test_zero_depth_at_range_boundary(oracle_lib):
    """O6 range test is inclusive at 0 and the key of depth 0 is the smallest
    (R4, R5): the plane z = x/64 - 1/8 (power-of-two slopes: exact) is 0.0
    exactly at the centres of column x = 8, where it beats an opaque earlier
    triangle at z = 2^-25 (primID 0); the depth written is +0.0 (sign bit clear;
    with IEEE round-to-nearest the plane cannot produce -0.0, so the key's
    0x7FFFFFFF mask is a guard that no input reaches).  Columns x < 8 are
    discarded (z < 0); at x = 9 z = 1/64 loses to 2^-25."""
    W = H = 64
    tris = [[(0.5, 0.5), (40.5, 0.5), (0.5, 40.5)], [(0.5, 0.5), (32.5, 0.5), (0.5, 32.5)]]
    zw = np.array([[2.0 ** -25] * 3, [-0.125, 0.375, -0.125]])
    v, i, m = pixel_scene(tris, zw, W, H)
    r = render(oracle_lib, v, i, m, W, H)
    d = r["depth"].view(np.uint32)
    for y in range(0, 20):
        assert r["primid"][y, 8] == 1 and d[y, 8] == 0, (y, r["primid"][y, 8], hex(d[y, 8]))
        assert r["primid"][y, 9] == 0 and r["depth"][y, 9] == np.float32(2.0 ** -25)
        assert (r["primid"][y, :8] == 0).all()  # B discarded there (z < 0)


# ------------------------------------------------------------------- depth ---
def test_constant_depth_is_exact(oracle_lib):
    """O6 closed form: a constant-z triangle (a = b = 0) gives z == zw0 at
    every covered pixel, and depth = 1.0 / primid = -1 on background (R6)."""
    v, i, m = pixel_scene([[(1.0, 2.0), (40.5, 5.0), (10.0, 60.25)]], 0.3125, 64, 64)
    r = render(oracle_lib, v, i, m, 64, 64)
    cov = r["covcount"] > 0
    assert cov.sum() > 500
    assert (r["depth"][cov] == np.float32(0.3125)).all()
    assert (r["depth"][~cov] == 1.0).all() and (r["primid"][~cov] == -1).all()
    assert (r["rgba"][~cov] == 0).all()


def test_sloped_depth_closed_form(oracle_lib):
    """O6 closed form: window depth zw = x/64 (power-of-two slope) on a
    triangle spanning the screen -> z at pixel centre = (x + 1/2)/64 exactly."""
    tri = [(0.0, 0.0), (64.0, 0.0), (0.0, 64.0)]
    zw = [[0.0, 1.0, 0.0]]
    v, i, m = pixel_scene([tri], zw, 64, 64)
    r = render(oracle_lib, v, i, m, 64, 64)
    ys, xs = np.nonzero(r["covcount"])
    assert len(xs) > 1500
    want = ((xs + 0.5) / 64.0).astype(np.float32)
    assert np.array_equal(r["depth"][ys, xs], want)


def test_depth_vs_exact_plane(oracle_lib):
    """O6 against the exact rational plane through the snapped corners: the
    fp32 depth is within 2e-6 (a few ulps of the terms) of the exact value."""
    from fractions import Fraction
    rng = np.random.default_rng(5)
    for _ in range(40):
        xy = np.stack([lattice(rng, 3, 0, 64, 1 / 256), lattice(rng, 3, 0, 64, 1 / 256)], 1)
        zw = lattice(rng, 3, 0.0, 1.0, 1 / 1024)
        v, i, m = pixel_scene([xy], [zw], 64, 64)
        r = render(oracle_lib, v, i, m, 64, 64)
        ys, xs = np.nonzero(r["primid"] >= 0)
        F = [(Fraction(float(a)), Fraction(float(b)), Fraction(float(z))) for (a, b), z in zip(xy, zw)]
        (x0, y0, z0), (x1, y1, z1), (x2, y2, z2) = F
        det = (x1 - x0) * (y2 - y0) - (x2 - x0) * (y1 - y0)
        if det == 0:
            continue
        for y, x in list(zip(ys, xs))[:50]:
            px, py = Fraction(2 * int(x) + 1, 2), Fraction(2 * int(y) + 1, 2)
            b1 = ((px - x0) * (y2 - y0) - (x2 - x0) * (py - y0)) / det
            b2 = ((x1 - x0) * (py - y0) - (px - x0) * (y1 - y0)) / det
            z = z0 + b1 * (z1 - z0) + b2 * (z2 - z0)
            assert abs(float(r["depth"][y, x]) - float(z)) <= 2e-6


def test_depth_range_discard(oracle_lib):
    """Per-pixel z in [0,1] discard (R3): a triangle at zw = 1.25 is covered but
    never drawn (alone: background); one at zw = -0.25 in front of zw = 0.5 is
    discarded (it would win the key comparison if kept); zw = 1.0 is kept."""
    tri = [(2.0, 2.0), (30.0, 4.0), (6.0, 28.0)]
    v, i, m = pixel_scene([tri], [[1.25] * 3], 32, 32)
    r = render(oracle_lib, v, i, m, 32, 32)
    assert r["covcount"].sum() > 300 and (r["primid"] == -1).all()
    v, i, m = pixel_scene([tri, tri], [[0.5] * 3, [-0.25] * 3], 32, 32)
    r = render(oracle_lib, v, i, m, 32, 32)
    cov = r["covcount"] > 0
    assert (r["primid"][cov] == 0).all() and (r["depth"][cov] == 0.5).all()
    v, i, m = pixel_scene([tri, tri], [[1.25] * 3, [1.0] * 3], 32, 32)
    r = render(oracle_lib, v, i, m, 32, 32)
    cov = r["covcount"] > 0
    assert (r["covcount"][cov] == 2).all()
    assert (r["primid"][cov] == 1).all() and (r["depth"][cov] == 1.0).all()


def test_tie_break_lower_primid_wins(oracle_lib):
    """two fragments at equal depth, primIDs 7 and 3 -> 3 wins
    (lexicographic (depth, primID) minimum, R5)."""
    rng = np.random.default_rng(6)
    tris, zs = [], []
    for t in range(8):
        if t in (3, 7):
            tris.append([(4.0, 4.0), (28.0, 6.0), (8.0, 28.0)])
            zs.append(0.5)
        else:
            xy = np.stack([lattice(rng, 3, 0, 32, 0.5), lattice(rng, 3, 0, 32, 0.5)], 1)
            tris.append(xy)
            zs.append(0.75)
    v, i, m = pixel_scene(tris, np.array(zs)[:, None].repeat(3, 1), 32, 32)
    r = render(oracle_lib, v, i, m, 32, 32)
    both = r["covcount"] > 0
    mask = np.zeros_like(both)
    t3 = pixel_scene([tris[3]], 0.5, 32, 32)
    mask = render(oracle_lib, *t3, 32, 32)["covcount"] > 0
    assert mask.sum() > 100
    assert (r["primid"][mask] == 3).all()


def test_merge_is_order_independent(oracle_lib):
    """permuting the triangle submission order gives the same
    depth image, and the same winner up to the relabelling wherever depths differ."""
    s = scenes.scene_soup(3000, 128, 128, seed=9, name="soup")
    r0 = render(oracle_lib, s.verts, s.idx, s.mvp, 128, 128)
    perm = np.random.default_rng(10).permutation(s.n_tris)
    r1 = render(oracle_lib, s.verts, s.idx[perm], s.mvp, 128, 128)
    assert np.array_equal(r0["depth"], r1["depth"])
    assert np.array_equal(r0["covcount"], r1["covcount"])
    fg = r0["primid"] >= 0
    assert np.array_equal(r0["primid"][fg], perm[r1["primid"][fg]])


# ----------------------------------------------------------------- shading ---
def test_lambert_listing1_values(oracle_lib):
    """PAPER.md:539-541 (Listing 1) values via tests/golden/lambert_values.txt."""
    for nx, ny, nz, r_, g_, b_ in load_golden("lambert_values.txt"):
        v, i, m = pixel_scene([[(0.0, 0.0), (32.0, 0.0), (0.0, 32.0)]], 0.5, 32, 32,
                              normals=[nx, ny, nz])
        r = render(oracle_lib, v, i, m, 32, 32)
        fg = r["primid"] >= 0
        assert np.abs(r["rgba"][fg] - np.array([r_, g_, b_, 1.0])).max() <= 1e-6


def test_perspective_correct_normal_vs_raycast(oracle_lib):
    """O7 perspective-correct interpolation pinned against an independent float64
    ray cast: unproject the pixel centre, intersect the object-space triangle,
    interpolate normals by object-space barycentrics, Lambert with Listing 1.
    A strongly slanted triangle (depth 1.5 .. 12) separates perspective-correct
    from screen-affine interpolation by far more than the tolerance."""
    W, H = 256, 192
    M = scenes.perspective_mvp()
    P = np.array([[-1.0, -0.8, -1.5], [1.2, -0.6, -1.6], [0.0, 2.0, -12.0]])
    N = np.array([[1.0, 0.0, 0.3], [0.0, 1.0, 0.3], [-0.6, -0.6, 1.0]])
    N /= np.linalg.norm(N, axis=1, keepdims=True)
    verts = scenes.pack_verts(P.astype(np.float32), N.astype(np.float32))
    idx = np.array([[0, 1, 2]], np.int32)
    r = render(oracle_lib, verts, idx, M, W, H)
    ys, xs = np.nonzero(r["primid"] == 0)
    assert len(xs) > 2000
    M64 = M.astype(np.float64).reshape(4, 4)
    Minv = np.linalg.inv(M64)
    L = np.array([1.0, 1.0, 1.0]) / math.sqrt(3)
    mat = np.array([0.80, 0.75, 0.65])
    P64 = P.astype(np.float32).astype(np.float64)
    N64 = N.astype(np.float32).astype(np.float64)
    n_tri = np.cross(P64[1] - P64[0], P64[2] - P64[0])
    err_pc, err_affine = [], []
    for y, x in zip(ys[::7], xs[::7]):
        ndc = np.array([(x + 0.5) / W * 2 - 1, 1 - (y + 0.5) / H * 2])
        a = Minv @ np.array([ndc[0], ndc[1], -1.0, 1.0])
        b = Minv @ np.array([ndc[0], ndc[1], 1.0, 1.0])
        a, b = a[:3] / a[3], b[:3] / b[3]
        d = b - a
        s = np.dot(n_tri, P64[0] - a) / np.dot(n_tri, d)
        q = a + s * d
        area = np.dot(np.cross(P64[1] - P64[0], P64[2] - P64[0]), n_tri)
        l1 = np.dot(np.cross(q - P64[0], P64[2] - P64[0]), n_tri) / area
        l2 = np.dot(np.cross(P64[1] - P64[0], q - P64[0]), n_tri) / area
        lam = np.array([1 - l1 - l2, l1, l2])
        n = lam @ N64
        want = mat * max(0.0, np.dot(n / np.linalg.norm(n), L))
        err_pc.append(np.abs(r["rgba"][y, x, :3] - want).max())
    assert max(err_pc) < 3e-3, max(err_pc)
    # the screen-affine alternative must be clearly worse (the pin has teeth)
    clip = np.concatenate([P64, np.ones((3, 1))], 1) @ M64.T
    scr = clip[:, :2] / clip[:, 3:4]
    for y, x in zip(ys[::7], xs[::7]):
        ndc = np.array([(x + 0.5) / W * 2 - 1, 1 - (y + 0.5) / H * 2])
        A = np.array([[scr[1, 0] - scr[0, 0], scr[2, 0] - scr[0, 0]],
                      [scr[1, 1] - scr[0, 1], scr[2, 1] - scr[0, 1]]])
        l1, l2 = np.linalg.solve(A, ndc - scr[0])
        n = np.array([1 - l1 - l2, l1, l2]) @ N64
        wrong = mat * max(0.0, np.dot(n / np.linalg.norm(n), L))
        err_affine.append(np.abs(r["rgba"][y, x, :3] - wrong).max())
    assert max(err_affine) > 10 * max(err_pc)


# -------------------------------------------------------------------- bins ---
def test_bins_nine_for_20px_box(oracle_lib):
    """bbox (0,0)-(20,20) with 8x8 bins -> the 3x3 block of bins."""
    v, i, m = pixel_scene([[(0.0, 0.0), (20.0, 0.0), (0.0, 20.0)]], 0.5, 64, 64)
    start, prims = oracle_lib.bins(v, i, m, 64, 64, 8, 8)
    nonempty = np.nonzero(np.diff(start))[0]
    assert sorted(nonempty.tolist()) == [0, 1, 2, 8, 9, 10, 16, 17, 18]
    assert (prims == 0).all()


@pytest.mark.parametrize("W,H,bw,bh", [(64, 64, 64, 64), (64, 64, 8, 8), (256, 256, 8, 8),
                                       (1024, 768, 8, 8), (100, 60, 16, 32)])
def test_bins_vs_bruteforce(oracle_lib, W, H, bw, bh):
    """SPEC.md:658 (1000 random boxes across grids incl. 1x1, 8x8, 32x32, 128x96):
    triangle t is in bin b iff some pixel of b (clipped to the screen) has its
    centre inside t's closed snapped bounding box (R11), brute-forced over bins;
    CSR order == numpy stable argsort of the primitive-ordered pairs."""
    rng = np.random.default_rng(W + bw)
    T = 1000
    ext = max(W, H)
    xy = np.stack([lattice(rng, 3 * T, -0.1 * ext, 1.1 * ext, 1 / 256),
                   lattice(rng, 3 * T, -0.1 * ext, 1.1 * ext, 1 / 256)], 1).reshape(T, 3, 2)
    # shrink half of them to small boxes (many single-bin and culled cases)
    small = rng.random(T) < 0.5
    xy[small] = xy[small][:, :1] + (xy[small] - xy[small][:, :1]) * 0.02
    xy = np.round(xy * 256) / 256
    v, i, m = pixel_scene(xy, 0.5, W, H)
    start, prims = oracle_lib.bins(v, i, m, W, H, bw, bh)
    binsX, binsY = -(-W // bw), -(-H // bh)
    pairs = []
    X = np.round(xy * 256).astype(np.int64)
    cx = np.arange(W) * 256 + 128          # every pixel centre, brute force
    cy = np.arange(H) * 256 + 128
    for t in range(T):
        area2 = (X[t, 1, 0] - X[t, 0, 0]) * (X[t, 2, 1] - X[t, 0, 1]) - \
                (X[t, 1, 1] - X[t, 0, 1]) * (X[t, 2, 0] - X[t, 0, 0])
        if area2 == 0:
            continue
        lo, hi = X[t].min(0), X[t].max(0)
        colhit = (cx >= lo[0]) & (cx <= hi[0])
        rowhit = (cy >= lo[1]) & (cy <= hi[1])
        bx_hit = np.add.reduceat(colhit.astype(int), np.arange(0, W, bw)) > 0
        by_hit = np.add.reduceat(rowhit.astype(int), np.arange(0, H, bh)) > 0
        for b in np.nonzero((by_hit[:, None] & bx_hit[None, :]).reshape(-1))[0]:
            pairs.append((b, t))
    pairs = np.array(pairs, np.int64).reshape(-1, 2)
    order = np.argsort(pairs[:, 0], kind="stable")
    want_prims = pairs[order, 1]
    want_start = np.searchsorted(pairs[order, 0], np.arange(binsX * binsY + 1))
    assert np.array_equal(prims, want_prims)
    assert np.array_equal(start, want_start)


def test_bins_rank_partition(oracle_lib):
    """Sort-first ownership (DirectMap round robin): the per-rank lists
    are the full lists restricted to bins b mod R == r; every bin exactly once."""
    s = scenes.scene_soup(2000, 256, 192, seed=13, name="soup", bin_sizes=(16,))
    full_s, full_p = oracle_lib.bins(s.verts, s.idx, s.mvp, 256, 192, 16, 16)
    NB = len(full_s) - 1
    for R in (2, 3, 4):
        seen = np.zeros(NB, np.int64)
        for rank in range(R):
            st, pr = oracle_lib.bins(s.verts, s.idx, s.mvp, 256, 192, 16, 16, rank, R)
            for b in range(NB):
                seg = pr[st[b]:st[b + 1]]
                if b % R == rank:
                    assert np.array_equal(seg, full_p[full_s[b]:full_s[b + 1]])
                    seen[b] += 1
                else:
                    assert len(seg) == 0
        assert (seen == 1).all()
