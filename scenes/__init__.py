"""Seeded synthetic scene generators shared by the oracle tests and the GPU path.

This module holds NO arithmetic of the method (no transform, snapping, binning,
coverage, depth or shading) -- only the input geometry, a camera matrix and a
light vector.  It is the one module both sides consume ("Inputs").

Scenes follow SURVEY.md section 8(d) (shapes of the paper's workloads,
PAPER.md:1241-1246 Fig. rastpics: Fairy Forest 174K tris "many small and large
triangles", Buddha 1.1M "very small triangles", all at 1024x768):

  c1  64x64, 8x8 bins, 16 triangles on a half-pixel lattice (oracle check)
  c2  1024x768, 16x16 bins, 100 UV spheres x 1000 tris  (Fairy-Forest scale)
  c3  1024x768, bins 8/16/32/64, one 1M-tri UV sphere    (Buddha scale)
  c4  1920x1080, 16x16 bins, 4M-tri random soup in NDC
  c5  3840x2160, 16x16 / 8x8 bins, 16M-tri jittered grid (micropolygon density)
  c6  1024x768, 32x32 bins, 256 bicubic Bezier patches (a bumpy height field in
      perspective) for the Reyes Split/Dice/Sample pipeline (
      SURVEY 8(f) NEXT-4); diced on the device into micropolygon quads (edge bound 2 px)

Layout: verts f32[V][8] = {px,py,pz,0, nx,ny,nz,0},
idx i32[T][3], mvp f32[16] row-major with clip = M * (x,y,z,1), light f32[3].
Seeds: config number (c1 -> 1, ...), numpy default_rng.
"""
from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field

import numpy as np

LIGHT = np.array([1.0, 1.0, 1.0], np.float32)  # Listing 1 lightvec


@dataclass
class Scene:
    name: str
    W: int
    H: int
    bin_sizes: tuple
    verts: np.ndarray
    idx: np.ndarray
    mvp: np.ndarray
    light: np.ndarray = field(default_factory=lambda: LIGHT.copy())

    @property
    def n_tris(self) -> int:
        return int(self.idx.shape[0])

    def sha256(self) -> str:
        h = hashlib.sha256()
        for a in (self.verts, self.idx, self.mvp, self.light):
            h.update(np.ascontiguousarray(a).tobytes())
        return h.hexdigest()


def pack_verts(pos, nrm) -> np.ndarray:
    """f32[V][8] from positions [V][3] and normals [V][3]."""
    V = pos.shape[0]
    v = np.zeros((V, 8), np.float32)
    v[:, 0:3] = pos
    v[:, 4:7] = nrm
    return v


def ortho_pixel_mvp(W: int, H: int) -> np.ndarray:
    """Ortho matrix mapping object (x, y) in pixels (y down) to NDC.

    For power-of-two W, H the viewport maps back to exactly (x, y)
    (SURVEY.md 8(c) pin for O1); object z = 2*zw - 1 gives window depth zw."""
    M = np.array([[2.0 / W, 0, 0, -1.0],
                  [0, -2.0 / H, 0, 1.0],
                  [0, 0, 1.0, 0],
                  [0, 0, 0, 1.0]], np.float64)
    return M.astype(np.float32).reshape(16)


def perspective_mvp(fovy_deg=60.0, aspect=4.0 / 3.0, near=0.1, far=100.0) -> np.ndarray:
    """OpenGL perspective projection (camera at origin looking down -z), row-major."""
    f = 1.0 / math.tan(math.radians(fovy_deg) / 2.0)
    M = np.array([[f / aspect, 0, 0, 0],
                  [0, f, 0, 0],
                  [0, 0, (far + near) / (near - far), 2 * far * near / (near - far)],
                  [0, 0, -1.0, 0]], np.float64)
    return M.astype(np.float32).reshape(16)


def random_unit(rng, n) -> np.ndarray:
    v = rng.normal(size=(n, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    return v.astype(np.float32)


# --------------------------------------------------------------------------
# UV sphere: L vertex rings x S slices + 2 poles; T = 2*S*L, V = S*L + 2
# --------------------------------------------------------------------------
def uv_sphere(L: int, S: int):
    """Unit UV sphere (poles on +-y): returns (unit positions f64[V][3], idx i64[T][3])."""
    theta = np.pi * (np.arange(L) + 1) / (L + 1)
    phi = 2 * np.pi * np.arange(S) / S
    st, ct = np.sin(theta)[:, None], np.cos(theta)[:, None]
    ring = np.stack([st * np.cos(phi)[None, :], np.broadcast_to(ct, (L, S)),
                     st * np.sin(phi)[None, :]], axis=-1).reshape(-1, 3)
    pos = np.concatenate([[[0.0, 1.0, 0.0]], ring, [[0.0, -1.0, 0.0]]], axis=0)
    top, bot = 0, S * L + 1
    r = lambda i, j: 1 + i * S + (j % S)  # noqa: E731
    j = np.arange(S)
    tris = [np.stack([np.full(S, top), r(0, j + 1), r(0, j)], 1)]
    i = np.arange(L - 1)[:, None]
    a, b, c, d = r(i, j), r(i + 1, j), r(i + 1, j + 1), r(i, j + 1)
    tris.append(np.stack([a, b, c], -1).reshape(-1, 3))
    tris.append(np.stack([a, c, d], -1).reshape(-1, 3))
    tris.append(np.stack([np.full(S, bot), r(L - 1, j), r(L - 1, j + 1)], 1))
    return pos, np.concatenate(tris, 0)


def scene_c1() -> Scene:
    """64x64, 8x8 bins, 16 triangles on a half-pixel lattice (oracle check).

    3 quads split on a diagonal (6 tris; quads A and B share an edge), a 6-tri
    fan around a vertex exactly on the pixel centre (32.5, 32.5), 4 free tris.
    Window depths from {0.25, 0.5, 0.75} with forced equal-depth overlaps.
    Random winding, random unit normals.  Object coords are pixel coords."""
    rng = np.random.default_rng(1)
    W = H = 64
    P = []   # positions (x, y, zw)
    tris = []

    def vert(x, y, zw):
        P.append((x, y, zw))
        return len(P) - 1

    # quads A, B (sharing edge x = 20), C; depths 0.5, 0.5, 0.25
    qa = [vert(4.5, 4.0, 0.5), vert(20.0, 4.0, 0.5), vert(20.0, 20.5, 0.5), vert(4.5, 20.5, 0.5)]
    qb = [qa[1], vert(36.0, 6.5, 0.5), vert(36.0, 22.0, 0.5), qa[2]]
    qc = [vert(40.5, 40.0, 0.25), vert(60.0, 41.5, 0.25), vert(58.5, 60.0, 0.25),
          vert(42.0, 58.5, 0.25)]
    for q in (qa, qb, qc):
        tris += [(q[0], q[1], q[2]), (q[0], q[2], q[3])]
    # fan of 6 around a vertex on the pixel centre (32.5, 32.5), depth 0.75
    c = vert(32.5, 32.5, 0.75)
    ring = [vert(32.5 + 6.0 * math.cos(a), 32.5 + 6.0 * math.sin(a), 0.75)
            for a in np.arange(6) * (2 * math.pi / 6)]
    # snap fan ring to the half-pixel lattice
    for k in ring:
        x, y, z = P[k]
        P[k] = (round(2 * x) / 2, round(2 * y) / 2, z)
    for k in range(6):
        tris.append((c, ring[k], ring[(k + 1) % 6]))
    # 4 free triangles: two equal-depth (0.5) overlapping quad A/B, one 0.25 over
    # the fan, one 0.75 spanning tile borders
    free = [((8.0, 8.5), (30.0, 12.0), (14.5, 26.0), 0.5),
            ((10.0, 2.5), (24.0, 16.0), (6.0, 18.0), 0.5),
            ((28.0, 28.0), (40.0, 30.5), (31.5, 42.0), 0.25),
            ((2.5, 44.0), (30.0, 48.0), (16.0, 63.5), 0.75)]
    for a, b, cc, z in free:
        tris.append((vert(*a, z), vert(*b, z), vert(*cc, z)))
    tris = np.array(tris, np.int64)
    # random winding per triangle
    for t in range(tris.shape[0]):
        if rng.random() < 0.5:
            tris[t, [1, 2]] = tris[t, [2, 1]]
    P = np.array(P, np.float64)
    pos = np.stack([P[:, 0], P[:, 1], 2.0 * P[:, 2] - 1.0], 1)
    verts = pack_verts(pos.astype(np.float32), random_unit(rng, P.shape[0]))
    return Scene("c1", W, H, (8,), verts, tris.astype(np.int32), ortho_pixel_mvp(W, H))


def scene_c2() -> Scene:
    """1024x768, 16x16 bins: 100 UV spheres of 20 rings x 25 slices (T=100,000,
    V=50,200), radii U[0.5,1.5], centres in the frustum at depth U[3,30]."""
    rng = np.random.default_rng(2)
    unit, tri = uv_sphere(20, 25)
    n = 100
    tanh = math.tan(math.radians(30.0))
    d = rng.uniform(3.0, 30.0, n)
    cx = rng.uniform(-0.8, 0.8, n) * d * tanh * (4.0 / 3.0)
    cy = rng.uniform(-0.8, 0.8, n) * d * tanh
    rad = rng.uniform(0.5, 1.5, n)
    pos = (unit[None] * rad[:, None, None] + np.stack([cx, cy, -d], 1)[:, None, :]).reshape(-1, 3)
    nrm = np.broadcast_to(unit[None], (n,) + unit.shape).reshape(-1, 3)
    idx = (tri[None] + (np.arange(n) * unit.shape[0])[:, None, None]).reshape(-1, 3)
    return Scene("c2", 1024, 768, (16,), pack_verts(pos.astype(np.float32), nrm.astype(np.float32)),
                 idx.astype(np.int32), perspective_mvp())


def scene_c3() -> Scene:
    """1024x768, bins 8/16/32/64: one UV sphere 500 rings x 1000 slices
    (T=1,000,000, V=500,002), radius 1 at distance 3.2 (~438 px wide)."""
    unit, tri = uv_sphere(500, 1000)
    pos = unit + np.array([0.0, 0.0, -3.2])
    return Scene("c3", 1024, 768, (8, 16, 32, 64),
                 pack_verts(pos.astype(np.float32), unit.astype(np.float32)),
                 tri.astype(np.int32), perspective_mvp())


def scene_soup(T: int, W: int, H: int, seed: int, name: str, bin_sizes=(16,)) -> Scene:
    """Random triangle soup in NDC (mvp = I): centres U([-1,1]^2), circumradius
    log-uniform [1,8] px, random vertex angles, z_ndc U[-0.8,0.8] +- 0.01."""
    rng = np.random.default_rng(seed)
    c = rng.uniform(-1.0, 1.0, (T, 2))
    r = np.exp(rng.uniform(math.log(1.0), math.log(8.0), T))
    ang = rng.uniform(0.0, 2 * math.pi, (T, 3))
    x = c[:, 0:1] + (r * 2.0 / W)[:, None] * np.cos(ang)
    y = c[:, 1:2] + (r * 2.0 / H)[:, None] * np.sin(ang)
    z = rng.uniform(-0.8, 0.8, (T, 1)) + rng.uniform(-0.01, 0.01, (T, 3))
    pos = np.stack([x, y, z], -1).reshape(-1, 3).astype(np.float32)
    nrm = random_unit(rng, 3 * T)
    idx = np.arange(3 * T, dtype=np.int32).reshape(T, 3)
    return Scene(name, W, H, bin_sizes, pack_verts(pos, nrm), idx, np.eye(4, dtype=np.float32).reshape(16))


def scene_fuzz(seed: int) -> Scene:
    """Randomised small case for differential testing (geometry only): random
    screen (1..300 px, odd sizes included) and bins, T in [0, 2500], and a mix
    of triangle kinds -- tiny, medium, screen-covering, slivers, degenerate
    (repeated corner), off-screen, beyond the guard band, behind the camera,
    non-finite corners, lattice-aligned shared edges with equal depths (ties),
    and vertex sharing (random index reuse)."""
    rng = np.random.default_rng(10_000 + seed)
    W, H = int(rng.integers(1, 301)), int(rng.integers(1, 301))
    if rng.random() < 0.3:
        W, H = int(rng.choice([16, 64, 128, 256])), int(rng.choice([16, 64, 128, 256]))
    bins = (int(rng.choice([8, 16, 32, 64])), int(rng.choice([8, 16, 32, 64])))
    T = int(rng.integers(0, 2501)) if rng.random() > 0.05 else 0
    pk = np.array([.30, .20, .05, .08, .04, .05, .04, .06, .03, .15])
    if rng.random() < 0.6:  # most cases without screen-covering triangles: background stays visible
        pk[2] = 0.0
    kind = rng.choice(10, size=T, p=pk / pk.sum())
    persp = rng.random() < 0.4
    # positions in NDC (identity mvp) or camera space in front of the camera (perspective)
    c = rng.uniform(-1.1, 1.1, (T, 2))
    px = np.array([2.0 / max(W, 1), 2.0 / max(H, 1)])
    rad = np.where(kind == 0, rng.uniform(0.2, 2.0, T),          # tiny (px)
          np.where(kind == 1, rng.uniform(2.0, 30.0, T),         # medium
          np.where(kind == 2, rng.uniform(200.0, 2000.0, T),     # covering / beyond screen
                   rng.uniform(1.0, 20.0, T))))
    ang = rng.uniform(0, 2 * math.pi, (T, 3))
    xy = c[:, None, :] + rad[:, None, None] * px[None, None, :] * np.stack([np.cos(ang), np.sin(ang)], -1)
    z = rng.uniform(-0.9, 0.9, (T, 1)) + rng.uniform(-0.05, 0.05, (T, 3))
    pos = np.concatenate([xy, z[..., None]], -1)                  # [T][3][3]
    sl = kind == 3                                                # slivers: corner 2 near edge 0-1
    pos[sl, 2, :2] = 0.5 * (pos[sl, 0, :2] + pos[sl, 1, :2]) + rng.normal(0, 1e-4, (sl.sum(), 2))
    dg = kind == 4                                                # degenerate: repeated corner
    pos[dg, 2] = pos[dg, 0]
    off = kind == 5                                               # off-screen
    pos[off, :, :2] += np.sign(rng.uniform(-1, 1, (off.sum(), 1, 2))) * 3.0
    gb = kind == 6                                                # beyond the guard band
    pos[gb, 0, :2] = rng.choice([-1, 1], (gb.sum(), 2)) * rng.uniform(1e4, 1e6, (gb.sum(), 2))
    lat = kind == 9                                               # half-pixel lattice, shared depth
    pos[lat, :, :2] = (np.round((pos[lat, :, :2] + 1) / px * 2) / 2) * px - 1
    pos[lat, :, 2] = 0.25
    if persp:   # NDC -> camera space at depth d with x, y scaled into the frustum
        d = rng.uniform(1.0, 20.0, (T, 1, 1))
        f = 1.0 / math.tan(math.radians(30.0))
        cam = np.concatenate([pos[..., :1] * d * (W / max(H, 1)) / f, pos[..., 1:2] * d / f,
                              -d + pos[..., 2:3] * 0.5], -1)
        beh = kind == 7                                           # behind the camera / straddling
        cam[beh, 0, 2] = rng.uniform(0.0, 5.0, beh.sum())
        pos = cam
    nf = kind == 8                                                # non-finite corner
    pos[nf, 1, rng.integers(0, 3)] = rng.choice([np.inf, -np.inf, np.nan])
    verts = pack_verts(pos.reshape(-1, 3).astype(np.float32), random_unit(rng, 3 * T))
    idx = np.arange(3 * T, dtype=np.int64).reshape(T, 3)
    if T > 1 and rng.random() < 0.5:                              # vertex sharing
        share = rng.random((T, 3)) < 0.2
        idx[share] = rng.integers(0, 3 * T, share.sum())
    mvp = perspective_mvp(aspect=W / max(H, 1)) if persp else np.eye(4, dtype=np.float32).reshape(16)
    light = random_unit(rng, 1)[0] if rng.random() < 0.5 else LIGHT.copy()
    return Scene(f"fuzz{seed}", W, H, bins, verts, idx.astype(np.int32), mvp, light)


def scene_c4(T: int = 4_000_000) -> Scene:
    """1920x1080, 16x16 bins, 4M-triangle random soup (sort-first case)."""
    return scene_soup(T, 1920, 1080, 4, "c4")


def scene_grid(nx: int, ny: int, W: int, H: int, seed: int, name: str, bin_sizes) -> Scene:
    """Jittered grid mesh over NDC [-1,1]^2: (nx+1)(ny+1) verts, 2*nx*ny tris,
    interior vertices jittered +-0.25 cell, alternating diagonals (a planar
    partition of the screen: every pixel centre is covered exactly once)."""
    rng = np.random.default_rng(seed)
    gx, gy = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1))  # [ny+1][nx+1]
    x = -1.0 + 2.0 * gx / nx
    y = -1.0 + 2.0 * gy / ny
    interior = (gx > 0) & (gx < nx) & (gy > 0) & (gy < ny)
    x = x + interior * rng.uniform(-0.25, 0.25, x.shape) * (2.0 / nx)
    y = y + interior * rng.uniform(-0.25, 0.25, y.shape) * (2.0 / ny)
    z = 0.5 + 0.1 * np.sin(3 * np.pi * x) * np.cos(2 * np.pi * y)
    pos = np.stack([x, y, z], -1).reshape(-1, 3).astype(np.float32)
    nrm = np.stack([-0.3 * np.cos(3 * np.pi * x), 0.2 * np.sin(2 * np.pi * y), np.ones_like(x)], -1)
    nrm = (nrm / np.linalg.norm(nrm, axis=-1, keepdims=True)).reshape(-1, 3).astype(np.float32)
    vid = lambda i, j: j * (nx + 1) + i  # noqa: E731
    i, j = np.meshgrid(np.arange(nx), np.arange(ny))
    a, b, c, d = vid(i, j), vid(i + 1, j), vid(i + 1, j + 1), vid(i, j + 1)
    alt = ((i + j) % 2 == 0)[..., None]
    t1 = np.where(alt, np.stack([a, b, c], -1), np.stack([a, b, d], -1))
    t2 = np.where(alt, np.stack([a, c, d], -1), np.stack([b, c, d], -1))
    idx = np.stack([t1, t2], 2).reshape(-1, 3).astype(np.int32)
    return Scene(name, W, H, bin_sizes, pack_verts(pos, nrm), idx, np.eye(4, dtype=np.float32).reshape(16))


def scene_c5() -> Scene:
    """3840x2160, 16M-triangle jittered grid (4000x2000 quads; V=8,006,001)."""
    return scene_grid(4000, 2000, 3840, 2160, 5, "c5", (16, 8))


@dataclass
class PatchScene:
    """Bicubic Bezier patches: f32[P][16][4], control point k = a*4 + b with a
    along u and b along v, (x, y, z, 0).  Diced on the device (Split/Dice)."""
    name: str
    W: int
    H: int
    bin_sizes: tuple
    patches: np.ndarray
    mvp: np.ndarray
    light: np.ndarray = field(default_factory=lambda: LIGHT.copy())
    dice_px: float = 2.0
    max_grid: int = 128

    @property
    def n_patches(self) -> int:
        return int(self.patches.shape[0])


def view_mvp(pitch_deg=25.0, eye_y=3.0, **persp) -> np.ndarray:
    """Perspective * view (camera at (0, eye_y, 0) pitched down), row-major."""
    c, s_ = math.cos(math.radians(pitch_deg)), math.sin(math.radians(pitch_deg))
    R = np.array([[1, 0, 0, 0], [0, c, -s_, 0], [0, s_, c, 0], [0, 0, 0, 1]], np.float64)
    T = np.eye(4)
    T[1, 3] = -eye_y
    P = perspective_mvp(**persp).astype(np.float64).reshape(4, 4)
    return (P @ R @ T).astype(np.float32).reshape(16)


def scene_patches(n: int = 16, seed: int = 6, W: int = 1024, H: int = 768, name: str = "c6",
                  x_range=(-6.0, 6.0), z_range=(-18.0, -3.0), dice_px: float = 2.0,
                  max_grid: int = 128) -> PatchScene:
    """n x n bicubic patches on a shared (3n+1)^2 control lattice (C0 across
    patch borders) over a bumpy height field y = h(x, z) in front of a
    camera pitched down (PAPER.md:1222-1225 Teapot/Bigguy are not shipped)."""
    rng = np.random.default_rng(seed)
    m = 3 * n + 1
    xs = np.linspace(*x_range, m)
    zs = np.linspace(*z_range, m)
    X, Z = np.meshgrid(xs, zs, indexing="ij")
    Y = 0.6 * np.sin(0.9 * X) * np.cos(0.7 * Z) + 0.3 * np.sin(2.1 * X + 1.3 * Z) + \
        rng.uniform(-0.15, 0.15, X.shape)
    lat = np.stack([X, Y, Z, np.zeros_like(X)], -1).astype(np.float32)
    patches = np.empty((n * n, 16, 4), np.float32)
    for pi in range(n):
        for pj in range(n):
            blk = lat[3 * pi:3 * pi + 4, 3 * pj:3 * pj + 4]   # [a (u)][b (v)]
            patches[pi * n + pj] = blk.reshape(16, 4)
    return PatchScene(name, W, H, (32,), patches, view_mvp(), dice_px=dice_px, max_grid=max_grid)


def scene_c6() -> PatchScene:
    return scene_patches()


CONFIGS = {"c1": scene_c1, "c2": scene_c2, "c3": scene_c3, "c4": scene_c4, "c5": scene_c5, "c6": scene_c6}


def make(name: str) -> Scene:
    return CONFIGS[name]()
