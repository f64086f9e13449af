"""Pins of the oracle's Reyes Split + Dice (R19-R21; PAPER.md:1172-1206,
SURVEY 8(f) NEXT-4) against closed forms and invariants (-m "not gpu").

None re-types the oracle's evaluation: the checks are the Bezier end-point
interpolation property, exact linear precision of the Bernstein basis on a
planar patch with power-of-two steps, the dice-rate closed form under the exact
ortho pixel matrix, and watertightness of the micropolygon mesh."""
from __future__ import annotations

import numpy as np

import scenes


def flat_patch(x0, z0, dx, dz, y=0.0):
    """Control point a*4+b = (x0 + a dx, y, z0 + b dz): a bilinear (planar) patch."""
    cp = np.zeros((16, 4), np.float32)
    for a in range(4):
        for b in range(4):
            cp[4 * a + b] = (x0 + a * dx, y, z0 + b * dz, 0)
    return cp


def test_corners_interpolate_control_points(oracle_lib):
    """A Bezier patch interpolates its 4 corner control points (u, v in {0, 1})."""
    s = scenes.scene_c6()
    G, verts, _ = oracle_lib.dice(s.patches[:8], s.mvp, s.W, s.H, s.dice_px, s.max_grid)
    vb = 0
    for p in range(8):
        gu, gv = G[p]
        P = verts[vb:vb + (gu + 1) * (gv + 1), :3].reshape(gu + 1, gv + 1, 3)
        cp = s.patches[p, :, :3].reshape(4, 4, 3)
        for (i, j), (a, b) in {(0, 0): (0, 0), (gu, 0): (3, 0), (0, gv): (0, 3), (gu, gv): (3, 3)}.items():
            assert np.array_equal(P[i, j], cp[a, b]), (p, i, j)
        vb += (gu + 1) * (gv + 1)


def test_planar_patch_linear_precision_and_normal(oracle_lib):
    """Linear precision: control points on a lattice with steps dx, dz give
    P(u, v) = (x0 + 3u dx, y, z0 + 3v dz) exactly (u = i/G, power-of-two G, all
    products exact), and the normal Pv x Pu = (0, 9 dx dz, 0) exactly."""
    W = H = 64
    M = scenes.ortho_pixel_mvp(W, H)
    # ortho maps x, y to pixels; this patch lies in the x-y plane (z = object depth)
    cp = np.zeros((16, 4), np.float32)
    for a in range(4):
        for b in range(4):
            cp[4 * a + b] = (4.0 + 8 * a, 2.0 + 4 * b, 0.0, 0)  # P = (4 + 24u, 2 + 12v, 0)
    G, verts, idx = oracle_lib.dice(cp[None], M, W, H, 2.0, 128)
    gu, gv = G[0]
    assert (gu, gv) == (16, 8)  # Lu = 24 px -> 16 x 2 >= 24 > 8 x 2;  Lv = 12 -> 8
    P = verts[:, :3].reshape(gu + 1, gv + 1, 3)
    u = np.arange(gu + 1)[:, None] / gu
    v = np.arange(gv + 1)[None, :] / gv
    assert np.array_equal(P[..., 0], np.broadcast_to(4 + 24 * u, P[..., 0].shape).astype(np.float32))
    assert np.array_equal(P[..., 1], np.broadcast_to(2 + 12 * v, P[..., 1].shape).astype(np.float32))
    assert (P[..., 2] == 0).all()
    # Pu = (24, 0, 0), Pv = (0, 12, 0): Pv x Pu = (0, 0, -288)
    n = verts[:, 4:7]
    assert (n[:, 0] == 0).all() and (n[:, 1] == 0).all() and (n[:, 2] == -288.0).all()
    assert idx.shape[0] == 2 * gu * gv and idx.max() == verts.shape[0] - 1


def test_dice_rate_closed_form(oracle_lib):
    """R19 under the exact ortho pixel matrix: control rows 10 px apart along u
    (polyline length 30 px) and 1 px along v (3 px): dice_px = 2 -> Gu = 16,
    Gv = 2; max_grid caps it; a control point behind the near plane (w <= eps)
    forces max_grid."""
    W = H = 256
    M = scenes.ortho_pixel_mvp(W, H)
    cp = np.zeros((16, 4), np.float32)
    for a in range(4):
        for b in range(4):
            cp[4 * a + b] = (20.0 + 10 * a, 30.0 + 1 * b, 0.0, 0)
    G, _, _ = oracle_lib.dice(cp[None], M, W, H, 2.0, 128)
    assert tuple(G[0]) == (16, 2)
    G, _, _ = oracle_lib.dice(cp[None], M, W, H, 2.0, 8)
    assert tuple(G[0]) == (8, 2)
    G, _, _ = oracle_lib.dice(cp[None], M, W, H, 0.25, 128)
    assert tuple(G[0]) == (128, 16)  # 30 / 0.25 = 120 -> 128;  3 / 0.25 = 12 -> 16
    P = scenes.perspective_mvp(aspect=1.0)
    cp2 = cp.copy()
    cp2[5, 2] = 1.0  # in front of the eye at z = +1: w = -1 <= eps
    G, _, _ = oracle_lib.dice(cp2[None], P, W, H, 2.0, 32)
    assert tuple(G[0]) == (32, 32)


def test_micropolygon_mesh_is_watertight(oracle_lib):
    """Two planar patches sharing a border (equal dice rates): their
    micropolygon meshes cover every pixel centre inside the union exactly once
    (shared border vertices are bit-identical: Bernstein end-point values)."""
    W = H = 64
    M = scenes.ortho_pixel_mvp(W, H)
    p0 = np.zeros((16, 4), np.float32)
    p1 = np.zeros((16, 4), np.float32)
    xs = [0.0, 5.0, 13.0, 18.0]  # uneven control spacing: a cubic parametrisation of a straight span
    for a in range(4):
        for b in range(4):
            p0[4 * a + b] = (6.0 + xs[a], 6.0 + 4 * b, 0.0, 0)
            p1[4 * a + b] = (6.0 + xs[a], 18.0 + 4 * b, 0.0, 0)
    pt = np.stack([p0, p1])
    G, verts, idx = oracle_lib.dice(pt, M, W, H, 1.0, 128)
    assert G[0][0] == G[1][0]  # same rate along the shared border (u)
    r = oracle_lib.render(verts, idx, M, np.ones(3, np.float32), W, H, want_covcount=True)
    cov = r["covcount"]
    assert cov.max() == 1
    # every pixel centre strictly inside the union [6, 24] x [6, 30] once
    assert cov[6:30, 6:24].min() == 1 and cov.sum() == 24 * 18
