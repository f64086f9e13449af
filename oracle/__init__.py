"""CPU oracle for the binned rasterizer (ctypes wrapper over piko_oracle.c).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product package ``paper_1404_6293_b200`` never imports it and
shares no code with it ("Oracle").

The C source follows SURVEY.md section 8(c) steps O1..O7 and cites PAPER.md
passages line by line; this wrapper only marshals numpy arrays.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "piko_oracle.c")
_LIB = os.path.join(_HERE, "libpiko_oracle.so")
_LIB_OMP = os.path.join(_HERE, "libpiko_oracle_omp.so")  # same source, -fopenmp (all host cores)

# -ffp-contract=off is mandatory: the op order (fmaf vs separate mul/add) is
# part of the definition the GPU path must reproduce bit for bit.
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c99", "-fPIC", "-shared"]

CLEAR_KEY = 0xFFFFFFFFFFFFFFFF


def build(force: bool = False) -> str:
    """Compile piko_oracle.c into libpiko_oracle.so (gcc; a checker, not the product).
    ORACLE_LIB overrides the library path (tools/oracle_mutations.py only)."""
    if os.environ.get("ORACLE_LIB"):
        return os.environ["ORACLE_LIB"]
    for lib, extra in ((_LIB, []), (_LIB_OMP, ["-fopenmp"])):
        if force or not os.path.exists(lib) or os.path.getmtime(lib) < os.path.getmtime(_SRC):
            tmp = lib + f".tmp{os.getpid()}"
            subprocess.check_call(["gcc", *CFLAGS, *extra, _SRC, "-o", tmp, "-lm"])
            os.replace(tmp, lib)
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        lib.oracle_setup.argtypes = [P, P, ctypes.c_int64, P, ctypes.c_int, ctypes.c_int, P, P]
        lib.oracle_setup.restype = ctypes.c_int
        lib.oracle_render.argtypes = [ctypes.c_int, ctypes.c_int, P, P, ctypes.c_int64, P, P,
                                      P, P, P, P, P]
        lib.oracle_render.restype = ctypes.c_int
        lib.oracle_bins.argtypes = [ctypes.c_int] * 6 + [P, P, ctypes.c_int64, P, P, P,
                                                          ctypes.c_int64]
        lib.oracle_bins.restype = ctypes.c_int64
        lib.oracle_dice_grid.argtypes = [P, ctypes.c_int64, P, ctypes.c_int, ctypes.c_int, ctypes.c_float,
                                         ctypes.c_int, P]
        lib.oracle_dice_grid.restype = ctypes.c_int
        lib.oracle_dice_mesh.argtypes = [P, ctypes.c_int64, P, P, P]
        lib.oracle_dice_mesh.restype = ctypes.c_int64
        _lib = lib
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _check_scene(verts, idx, mvp):
    verts = np.ascontiguousarray(verts, dtype=np.float32)
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    mvp = np.ascontiguousarray(np.asarray(mvp, dtype=np.float32).reshape(16))
    assert verts.ndim == 2 and verts.shape[1] == 8, "verts must be f32[V][8]"
    assert idx.ndim == 2 and idx.shape[1] == 3, "idx must be i32[T][3]"
    if idx.size:
        assert idx.min() >= 0 and idx.max() < verts.shape[0], "idx out of range"
    return verts, idx, mvp


def setup(verts, idx, mvp, W, H):
    """Per-triangle O1..O4 record: (ints[T][12], floats[T][6]); see piko_oracle.c."""
    verts, idx, mvp = _check_scene(verts, idx, mvp)
    T = idx.shape[0]
    oi = np.zeros((T, 12), np.int32)
    of = np.zeros((T, 6), np.float32)
    _load().oracle_setup(_ptr(verts), _ptr(idx), T, _ptr(mvp), W, H, _ptr(oi), _ptr(of))
    return oi, of


def render(verts, idx, mvp, light, W, H, want_covcount=False, want_keys=False):
    """Full frame.  Returns dict rgba f32[H][W][4], depth f32[H][W], primid i32[H][W]
    (+ covcount u32[H][W], keys u64[H][W] on request)."""
    verts, idx, mvp = _check_scene(verts, idx, mvp)
    light = np.ascontiguousarray(np.asarray(light, np.float32).reshape(3))
    rgba = np.empty((H, W, 4), np.float32)
    depth = np.empty((H, W), np.float32)
    primid = np.empty((H, W), np.int32)
    cov = np.empty((H, W), np.uint32) if want_covcount else None
    keys = np.empty((H, W), np.uint64) if want_keys else None
    rc = _load().oracle_render(W, H, _ptr(verts), _ptr(idx), idx.shape[0], _ptr(mvp),
                               _ptr(light), _ptr(rgba), _ptr(depth), _ptr(primid), _ptr(cov),
                               _ptr(keys))
    if rc != 0:
        raise ValueError(f"oracle_render failed rc={rc}")
    out = {"rgba": rgba, "depth": depth, "primid": primid}
    if want_covcount:
        out["covcount"] = cov
    if want_keys:
        out["keys"] = keys
    return out


def dice(patches, mvp, W, H, dice_px, max_grid):
    """Reyes Split + Dice (R19-R21): per-patch dice rates G i32[P][2]
    = (Gu, Gv) and the micropolygon mesh (verts f32[V][8], idx i32[T][3]) in
    patch order."""
    patches = np.ascontiguousarray(patches, dtype=np.float32).reshape(-1, 16, 4)
    mvp = np.ascontiguousarray(np.asarray(mvp, dtype=np.float32).reshape(16))
    n = patches.shape[0]
    G = np.zeros((n, 2), np.int32)
    lib = _load()
    lib.oracle_dice_grid(_ptr(patches), n, _ptr(mvp), W, H, float(dice_px), int(max_grid), _ptr(G))
    g = G.astype(np.int64)
    V, T = int(((g[:, 0] + 1) * (g[:, 1] + 1)).sum()), int((2 * g[:, 0] * g[:, 1]).sum())
    verts = np.zeros((V, 8), np.float32)
    idx = np.zeros((T, 3), np.int32)
    got = lib.oracle_dice_mesh(_ptr(patches), n, _ptr(G), _ptr(verts), _ptr(idx))
    assert got == T
    return G, verts, idx


_lib_omp = None


def render_mt(verts, idx, mvp, light, W, H):
    """render() on all host cores (OpenMP over row bands; byte-identical).
    Returns (frame dict, threads used)."""
    global _lib_omp
    if _lib_omp is None:
        build()
        lib = ctypes.CDLL(_LIB_OMP)
        P = ctypes.c_void_p
        lib.oracle_render_mt.argtypes = [ctypes.c_int, ctypes.c_int, P, P, ctypes.c_int64, P, P, P, P, P]
        lib.oracle_render_mt.restype = ctypes.c_int
        _lib_omp = lib
    verts, idx, mvp = _check_scene(verts, idx, mvp)
    light = np.ascontiguousarray(np.asarray(light, np.float32).reshape(3))
    rgba = np.empty((H, W, 4), np.float32)
    depth = np.empty((H, W), np.float32)
    primid = np.empty((H, W), np.int32)
    n = _lib_omp.oracle_render_mt(W, H, _ptr(verts), _ptr(idx), idx.shape[0], _ptr(mvp), _ptr(light),
                                  _ptr(rgba), _ptr(depth), _ptr(primid))
    if n < 0:
        raise ValueError(f"oracle_render_mt failed rc={n}")
    return {"rgba": rgba, "depth": depth, "primid": primid}, n


def bins(verts, idx, mvp, W, H, bin_w, bin_h, rank=0, nranks=1):
    """Bin CSR (bin_start i32[NB+1], bin_prims i32[P]) in primitive order."""
    verts, idx, mvp = _check_scene(verts, idx, mvp)
    NB = ((W + bin_w - 1) // bin_w) * ((H + bin_h - 1) // bin_h)
    start = np.zeros(NB + 1, np.int32)
    cap = max(1024, 2 * idx.shape[0])
    lib = _load()
    while True:
        prims = np.zeros(cap, np.int32)
        P = lib.oracle_bins(W, H, bin_w, bin_h, rank, nranks, _ptr(verts), _ptr(idx),
                            idx.shape[0], _ptr(mvp), _ptr(start), _ptr(prims), cap)
        if P < 0:
            raise MemoryError("oracle_bins allocation failed")
        if P <= cap:
            return start, prims[:P].copy()
        cap = int(P)
