"""Shared test helpers: tiny hand-built scenes and independent exact checks.

Nothing here implements the method: the coverage check below is an
independently formulated definition (Cramer's-rule barycentrics of an
infinitesimally perturbed sample point, in exact rationals), used to pin the
oracle's integer edge-function + top-left formulation (R1).
"""
from __future__ import annotations

import os
from fractions import Fraction

import numpy as np

import scenes

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_golden(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append([float(v) for v in line.split()])
    return np.array(rows)


def pixel_scene(tris_xy, zw, W, H, normals=None):
    """Triangles given in pixel coordinates (x, y) with window depth zw per
    triangle (scalar) or per corner; ortho pixel mvp (exact for power-of-two W,H)."""
    tris_xy = np.asarray(tris_xy, np.float64).reshape(-1, 3, 2)
    T = tris_xy.shape[0]
    zw = np.asarray(zw, np.float64)
    zw = np.broadcast_to(zw.reshape(-1, 1) if zw.ndim <= 1 and zw.size in (1, T) else zw, (T, 3))
    pos = np.concatenate([tris_xy, (2.0 * zw - 1.0)[..., None]], -1).reshape(-1, 3)
    if normals is None:
        nrm = np.tile(np.array([0.0, 0.0, 1.0]), (3 * T, 1))
    else:
        nrm = np.broadcast_to(np.asarray(normals, np.float64).reshape(-1, 3), (3 * T, 3))
    verts = scenes.pack_verts(pos.astype(np.float32), nrm.astype(np.float32))
    idx = np.arange(3 * T, dtype=np.int32).reshape(T, 3)
    return verts, idx, scenes.ortho_pixel_mvp(W, H)


_DELTA = Fraction(1, 2 ** 40)


def covered_exact(tri_xy, x, y):
    """Is the centre of pixel (x, y) inside the triangle, by the perturbed-point
    definition: sample at (x + 1/2 + d, y + 1/2 + d^2) for an infinitesimal d
    (here d = 2^-40, exact for vertices on the 1/256 lattice within +-2^12 px),
    strictly inside by Cramer's-rule barycentric coordinates (any winding)."""
    (x0, y0), (x1, y1), (x2, y2) = [(Fraction(a), Fraction(b)) for a, b in tri_xy]
    px = Fraction(2 * x + 1, 2) + _DELTA
    py = Fraction(2 * y + 1, 2) + _DELTA * _DELTA
    det = (x1 - x0) * (y2 - y0) - (x2 - x0) * (y1 - y0)
    if det == 0:
        return False
    b1 = ((px - x0) * (y2 - y0) - (x2 - x0) * (py - y0)) / det
    b2 = ((x1 - x0) * (py - y0) - (px - x0) * (y1 - y0)) / det
    b0 = 1 - b1 - b2
    return b0 > 0 and b1 > 0 and b2 > 0


def lattice(rng, n, lo, hi, step):
    """n random values on the lattice step*k within [lo, hi]."""
    k = rng.integers(int(np.ceil(lo / step)), int(np.floor(hi / step)) + 1, n)
    return k * step
