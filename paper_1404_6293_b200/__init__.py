"""B200-native binned triangle rasterizer (Piko, arXiv 1404.6293) -- Python binding.

A thin ctypes binding over ``libpiko.so`` (the C ABI of ``include/piko.h``):
argument marshalling only -- every step of the path (vertex transform, setup,
AssignBin count / scan / stable scatter, Schedule, per-bin Process, shading,
write-back, NCCL tile gather) runs in the CUDA kernels of ``csrc/``.  PyTorch
is used for device memory, streams and process groups.  There is no CPU
fallback: importing this package without the built library raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpiko.so")

PIKO_OK, PIKO_EINVAL, PIKO_ENOMEM, PIKO_ECUDA, PIKO_ENCCL, PIKO_ECAPACITY, PIKO_ESTATE = 0, -1, -2, -3, -4, -5, -6
PIKO_DEBUG_COVERAGE_COUNT = 1
PIKO_SYNC_CHECKED, PIKO_SYNC_ASYNC = 0, 1
PIKO_PIPE_BINNED, PIKO_PIPE_FREEPIPE, PIKO_PIPE_BASELINE = 0, 1, 2
PIKO_MAX_SHADER_ITERS = 1 << 20
PIKO_MULTI_SORT_FIRST, PIKO_MULTI_SORT_LAST = 0, 1
PIKO_XPORT_NCCL, PIKO_XPORT_P2P = 0, 1

# names of every symbol include/piko.h declares (checked by tests)
EXPORTS = ("piko_create", "piko_draw", "piko_draw_host", "piko_draw_host_async", "piko_finish", "piko_set_sync",
           "piko_destroy", "piko_last_error", "piko_get_primid", "piko_get_bins",
           "piko_set_debug", "piko_get_coverage", "piko_set_partition", "piko_attach_comm",
           "piko_get_stats", "piko_nccl_unique_id", "piko_draw_indexed",
           "piko_draw_tile_keys", "piko_resolve_keys", "piko_tile_keys_count", "piko_owned_bins",
           "piko_set_pipeline", "piko_set_profiling", "piko_get_profile", "piko_set_multi",
           "piko_triangle_range", "piko_set_transport", "piko_attach_local_peers",
           "piko_p2p_export", "piko_p2p_import", "piko_set_shader_cost", "piko_draw_patches",
           "piko_get_diced")
STAGES = ("clear", "vertex", "setup", "expand", "sort", "tile", "gather", "resolve")


class PikoError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"piko error {code}: {msg}")
        self.code = code


class piko_stats(ctypes.Structure):
    _fields_ = [("n_tris", ctypes.c_int64), ("n_live", ctypes.c_int64),
                ("n_pairs", ctypes.c_int64), ("n_bins", ctypes.c_int64),
                ("owned_bins", ctypes.c_int64), ("pair_capacity", ctypes.c_int64),
                ("radix_passes", ctypes.c_int32), ("kernels_per_frame", ctypes.c_int32),
                ("assign_mode", ctypes.c_int32), ("reserved", ctypes.c_int32), ("cm_rows", ctypes.c_int64)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build() "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P, I, I64, U = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint
    sig = {
        "piko_create": ([I, I, I, I], P),
        "piko_draw": ([P, P, P, ctypes.c_int32, P, P, P, P, P], I),
        "piko_draw_host": ([P, P, I64, P, ctypes.c_int32, P, P, P, P, P], I),
        "piko_draw_host_async": ([P, P, I64, P, ctypes.c_int32, P, P, P, P, P], I),
        "piko_draw_indexed": ([P, P, I64, P, ctypes.c_int32, P, P, P, P, P], I),
        "piko_draw_tile_keys": ([P, P, I64, P, ctypes.c_int32, P, P, P, P], I),
        "piko_resolve_keys": ([P, P, I64, P, ctypes.c_int32, P, P, I, P, P, P, P], I),
        "piko_tile_keys_count": ([P], I64),
        "piko_owned_bins": ([I, I, I, I, I, I, P, I64], I64),
        "piko_set_pipeline": ([P, I], I),
        "piko_set_shader_cost": ([P, I, I], I),
        "piko_finish": ([P], I),
        "piko_set_sync": ([P, I], I),
        "piko_destroy": ([P], None),
        "piko_last_error": ([P], ctypes.c_char_p),
        "piko_get_primid": ([P, ctypes.POINTER(P)], I),
        "piko_get_bins": ([P, ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(I64)], I),
        "piko_set_debug": ([P, U], I),
        "piko_get_coverage": ([P, ctypes.POINTER(P)], I),
        "piko_set_partition": ([P, I, I], I),
        "piko_set_multi": ([P, I], I),
        "piko_set_transport": ([P, I], I),
        "piko_attach_local_peers": ([P, P, I, I], I),
        "piko_p2p_export": ([P, I, P], I),
        "piko_p2p_import": ([P, P, I, I], I),
        "piko_triangle_range": ([I64, I, I, ctypes.POINTER(I64), ctypes.POINTER(I64)], I),
        "piko_attach_comm": ([P, P, I, I], I),
        "piko_get_stats": ([P, ctypes.POINTER(piko_stats)], I),
        "piko_nccl_unique_id": ([P], I),
        "piko_set_profiling": ([P, I], I),
        "piko_get_profile": ([P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(I64)], I),
        "piko_draw_patches": ([P, P, ctypes.c_int32, P, P, ctypes.c_float, ctypes.c_int32, P, P, P], I),
        "piko_get_diced": ([P, ctypes.POINTER(P), ctypes.POINTER(I64), ctypes.POINTER(P), ctypes.POINTER(I64)], I),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes, f.restype = args, res
    return lib


_lib = _load()
lib = _lib


def _f32x(vals, n):
    arr = (ctypes.c_float * n)(*[float(v) for v in vals])
    return arr


def _dev_ptr(t, dtype, name):
    import torch
    if t is None:
        return None
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch tensor")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype or not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous {dtype}")
    return ctypes.c_void_p(t.data_ptr())


def _stream_ptr(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _check(ctx, rc):
    if rc != PIKO_OK:
        raise PikoError(rc, piko_last_error(ctx))
    return rc


# ---- the C ABI, one Python function per entry point -------------------------
_dims = {}  # ctx handle -> (width, height): shape checks of the output buffers


def piko_create(width, height, bin_w, bin_h):
    h = _lib.piko_create(width, height, bin_w, bin_h)
    if not h:
        raise PikoError(PIKO_EINVAL, _lib.piko_last_error(None).decode())
    _dims[h] = (width, height)
    return ctypes.c_void_p(h)


def _check_scene(verts, idx, n_tris=None):
    """verts f32[V][8], idx i32[T][3] (n_tris <= T): the C ABI reads them raw."""
    if verts is not None and (verts.dim() != 2 or verts.shape[1] != 8):
        raise ValueError(f"verts must be [V][8], got {tuple(verts.shape)}")
    if idx is not None:
        if idx.dim() != 2 or idx.shape[1] != 3:
            raise ValueError(f"idx must be [T][3], got {tuple(idx.shape)}")
        if n_tris is not None and int(n_tris) > idx.shape[0]:
            raise ValueError(f"n_tris {n_tris} > idx rows {idx.shape[0]}")


def _check_outputs(ctx, rgba, depth):
    W, H = _dims.get(ctx.value, (None, None))
    if W is None:
        return
    if rgba is not None and rgba.numel() < 4 * W * H:
        raise ValueError(f"out_rgba holds {rgba.numel()} floats, need {4 * W * H} (H x W x 4)")
    if depth is not None and depth.numel() < W * H:
        raise ValueError(f"out_depth holds {depth.numel()} floats, need {W * H} (H x W)")


def piko_destroy(ctx):
    _dims.pop(ctx.value, None)
    _lib.piko_destroy(ctx)


def piko_last_error(ctx):
    m = _lib.piko_last_error(ctx)
    return m.decode() if m else ""


def piko_draw(ctx, verts, idx, n_tris, mvp, light, out_rgba, out_depth, stream=None, check=True):
    import torch
    _check_scene(verts, idx, n_tris)
    _check_outputs(ctx, out_rgba, out_depth)
    rc = _lib.piko_draw(ctx, _dev_ptr(verts, torch.float32, "verts"),
                        _dev_ptr(idx, torch.int32, "idx"), int(n_tris), _f32x(mvp, 16),
                        _f32x(light, 3), _dev_ptr(out_rgba, torch.float32, "out_rgba"),
                        _dev_ptr(out_depth, torch.float32, "out_depth"), _stream_ptr(stream))
    return _check(ctx, rc) if check else rc


def piko_draw_indexed(ctx, verts, n_verts, idx, n_tris, mvp, light, out_rgba, out_depth,
                      stream=None, check=True):
    import torch
    _check_scene(verts, idx, n_tris)
    if verts is not None and int(n_verts) > verts.shape[0]:
        raise ValueError(f"n_verts {n_verts} > verts rows {verts.shape[0]}")
    _check_outputs(ctx, out_rgba, out_depth)
    rc = _lib.piko_draw_indexed(ctx, _dev_ptr(verts, torch.float32, "verts"), int(n_verts),
                                _dev_ptr(idx, torch.int32, "idx"), int(n_tris), _f32x(mvp, 16),
                                _f32x(light, 3), _dev_ptr(out_rgba, torch.float32, "out_rgba"),
                                _dev_ptr(out_depth, torch.float32, "out_depth"), _stream_ptr(stream))
    return _check(ctx, rc) if check else rc


def piko_owned_bins(width, height, bin_w, bin_h, rank, nranks):
    """Owned bins of a rank in sort-first payload order (host-only, no CUDA)."""
    import numpy as np
    n = _lib.piko_owned_bins(width, height, bin_w, bin_h, rank, nranks, None, 0)
    if n < 0:
        raise PikoError(int(n), "bad arguments")
    out = np.zeros(max(int(n), 1), np.int32)
    _lib.piko_owned_bins(width, height, bin_w, bin_h, rank, nranks,
                         out.ctypes.data_as(ctypes.c_void_p), int(n))
    return out[:n]


def piko_tile_keys_count(ctx):
    return int(_lib.piko_tile_keys_count(ctx))


def piko_draw_tile_keys(ctx, verts, idx, mvp, light, tile_keys, stream=None):
    """This rank's owned bins as packed u64 tile keys (the sort-first payload)."""
    import torch
    rc = _lib.piko_draw_tile_keys(ctx, _dev_ptr(verts, torch.float32, "verts"), verts.shape[0],
                                  _dev_ptr(idx, torch.int32, "idx"), idx.shape[0], _f32x(mvp, 16),
                                  _f32x(light, 3), _dev_ptr(tile_keys, torch.int64, "tile_keys"),
                                  _stream_ptr(stream))
    return _check(ctx, rc)


def piko_resolve_keys(ctx, verts, idx, mvp, light, nranks, all_keys, out_rgba, out_depth, stream=None):
    """Rank 0's resolve of gathered tile keys (u64[nranks][owned_max][bw*bh])."""
    import torch
    rc = _lib.piko_resolve_keys(ctx, _dev_ptr(verts, torch.float32, "verts"), verts.shape[0],
                                _dev_ptr(idx, torch.int32, "idx"), idx.shape[0], _f32x(mvp, 16),
                                _f32x(light, 3), int(nranks),
                                _dev_ptr(all_keys, torch.int64, "all_keys"),
                                _dev_ptr(out_rgba, torch.float32, "out_rgba"),
                                _dev_ptr(out_depth, torch.float32, "out_depth"), _stream_ptr(stream))
    return _check(ctx, rc)


def piko_draw_host(ctx, verts, idx, mvp, light, out_rgba, out_depth, stream=None):
    """verts/idx/out_* are CPU torch tensors (pinned for full bandwidth)."""
    import torch
    for t in (verts, idx, out_rgba, out_depth):
        if t.is_cuda or not t.is_contiguous():
            raise ValueError("piko_draw_host takes contiguous CPU tensors")
    for t, dt, name in ((verts, torch.float32, "verts"), (idx, torch.int32, "idx"),
                        (out_rgba, torch.float32, "out_rgba"), (out_depth, torch.float32, "out_depth")):
        if t.dtype != dt:
            raise ValueError(f"{name} must be {dt}")
    _check_scene(verts, idx)
    _check_outputs(ctx, out_rgba, out_depth)
    rc = _lib.piko_draw_host(ctx, ctypes.c_void_p(verts.data_ptr()), verts.shape[0],
                             ctypes.c_void_p(idx.data_ptr()), idx.shape[0], _f32x(mvp, 16),
                             _f32x(light, 3), ctypes.c_void_p(out_rgba.data_ptr()),
                             ctypes.c_void_p(out_depth.data_ptr()), _stream_ptr(stream))
    return _check(ctx, rc)


def piko_draw_host_async(ctx, verts, idx, mvp, light, out_rgba, out_depth, stream=None):
    """Pipelined piko_draw_host: enqueues upload, draw and download and returns
    (pinned CPU tensors; read the outputs after synchronising `stream` or
    piko_finish).  Errors are asynchronous (reported by a later call / finish)."""
    import torch
    for t in (verts, idx, out_rgba, out_depth):
        if t.is_cuda or not t.is_contiguous():
            raise ValueError("piko_draw_host_async takes contiguous CPU tensors")
    for t, dt, name in ((verts, torch.float32, "verts"), (idx, torch.int32, "idx"),
                        (out_rgba, torch.float32, "out_rgba"), (out_depth, torch.float32, "out_depth")):
        if t.dtype != dt:
            raise ValueError(f"{name} must be {dt}")
    _check_scene(verts, idx)
    _check_outputs(ctx, out_rgba, out_depth)
    rc = _lib.piko_draw_host_async(ctx, ctypes.c_void_p(verts.data_ptr()), verts.shape[0],
                                   ctypes.c_void_p(idx.data_ptr()), idx.shape[0], _f32x(mvp, 16),
                                   _f32x(light, 3), ctypes.c_void_p(out_rgba.data_ptr()),
                                   ctypes.c_void_p(out_depth.data_ptr()), _stream_ptr(stream))
    return _check(ctx, rc)


def piko_draw_patches(ctx, patches, mvp, light, dice_px, max_grid, out_rgba, out_depth, stream=None,
                      check=True):
    """Reyes: Split/Dice the bicubic patches (f32[P][16][4] CUDA tensor) on the
    device and draw the micropolygons (NEXT-4)."""
    import torch
    if patches.dim() != 3 or tuple(patches.shape[1:]) != (16, 4):
        raise ValueError(f"patches must be [P][16][4], got {tuple(patches.shape)}")
    _check_outputs(ctx, out_rgba, out_depth)
    rc = _lib.piko_draw_patches(ctx, _dev_ptr(patches, torch.float32, "patches"), int(patches.shape[0]),
                                _f32x(mvp, 16), _f32x(light, 3), ctypes.c_float(dice_px), int(max_grid),
                                _dev_ptr(out_rgba, torch.float32, "out_rgba"),
                                _dev_ptr(out_depth, torch.float32, "out_depth"), _stream_ptr(stream))
    return _check(ctx, rc) if check else rc


def piko_get_diced(ctx):
    """(verts ptr, n_verts, idx ptr, n_tris) of the last piko_draw_patches mesh."""
    v, i = ctypes.c_void_p(), ctypes.c_void_p()
    nv, nt = ctypes.c_int64(), ctypes.c_int64()
    _check(ctx, _lib.piko_get_diced(ctx, ctypes.byref(v), ctypes.byref(nv), ctypes.byref(i), ctypes.byref(nt)))
    return v.value, nv.value, i.value, nt.value


def piko_finish(ctx):
    return _lib.piko_finish(ctx)


def piko_set_sync(ctx, mode):
    return _check(ctx, _lib.piko_set_sync(ctx, mode))


def piko_set_pipeline(ctx, pipeline):
    return _check(ctx, _lib.piko_set_pipeline(ctx, pipeline))


def piko_set_shader_cost(ctx, iters, forward):
    return _check(ctx, _lib.piko_set_shader_cost(ctx, iters, forward))


def piko_get_primid(ctx):
    p = ctypes.c_void_p()
    _check(ctx, _lib.piko_get_primid(ctx, ctypes.byref(p)))
    return p.value


def piko_get_bins(ctx):
    s, q, n = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_int64()
    _check(ctx, _lib.piko_get_bins(ctx, ctypes.byref(s), ctypes.byref(q), ctypes.byref(n)))
    return s.value, q.value, n.value


def piko_set_debug(ctx, flags):
    return _check(ctx, _lib.piko_set_debug(ctx, flags))


def piko_get_coverage(ctx):
    p = ctypes.c_void_p()
    _check(ctx, _lib.piko_get_coverage(ctx, ctypes.byref(p)))
    return p.value


def piko_set_partition(ctx, rank, nranks):
    return _check(ctx, _lib.piko_set_partition(ctx, rank, nranks))


def piko_set_multi(ctx, mode):
    return _check(ctx, _lib.piko_set_multi(ctx, mode))


def piko_set_transport(ctx, transport):
    return _check(ctx, _lib.piko_set_transport(ctx, transport))


def piko_attach_local_peers(ctx, root, rank, nranks):
    return _check(ctx, _lib.piko_attach_local_peers(ctx, root, rank, nranks))


def piko_p2p_export(ctx, nranks) -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(ctx, _lib.piko_p2p_export(ctx, nranks, buf))
    return buf.raw


def piko_p2p_import(ctx, handles: bytes, rank, nranks):
    buf = ctypes.create_string_buffer(bytes(handles), 128)
    return _check(ctx, _lib.piko_p2p_import(ctx, buf, rank, nranks))


def piko_triangle_range(n_tris, rank, nranks):
    """Sort-last triangle range (t0, t1) of a rank (host-only, no CUDA)."""
    t0, t1 = ctypes.c_int64(), ctypes.c_int64()
    rc = _lib.piko_triangle_range(int(n_tris), rank, nranks, ctypes.byref(t0), ctypes.byref(t1))
    if rc != PIKO_OK:
        raise PikoError(rc, "bad arguments")
    return t0.value, t1.value


def piko_attach_comm(ctx, unique_id: bytes, rank, nranks):
    buf = ctypes.create_string_buffer(bytes(unique_id), 128)
    return _check(ctx, _lib.piko_attach_comm(ctx, buf, rank, nranks))


def piko_get_stats(ctx):
    st = piko_stats()
    _check(ctx, _lib.piko_get_stats(ctx, ctypes.byref(st)))
    return {f: getattr(st, f) for f, _ in piko_stats._fields_}


def piko_nccl_unique_id():
    buf = ctypes.create_string_buffer(128)
    rc = _lib.piko_nccl_unique_id(buf)
    if rc != PIKO_OK:
        raise PikoError(rc, _lib.piko_last_error(None).decode())
    return buf.raw


def piko_set_profiling(ctx, on):
    return _check(ctx, _lib.piko_set_profiling(ctx, int(bool(on))))


def piko_get_profile(ctx):
    """{stage: total ms} and the number of profiled frames."""
    ms = (ctypes.c_double * len(STAGES))()
    n = ctypes.c_int64()
    _check(ctx, _lib.piko_get_profile(ctx, ms, ctypes.byref(n)))
    return dict(zip(STAGES, list(ms))), n.value


# ---- convenience wrapper ------------------------------------------------------
class Renderer:
    """Owns a piko_ctx plus torch output buffers for one framebuffer shape."""

    def __init__(self, width, height, bin_w=16, bin_h=None, device=None, sync="checked"):
        """sync="checked" (this wrapper's default): every draw waits for its
        frame and regrows + re-issues on a capacity miss, so the frame read
        afterwards is always valid; "async" keeps the C ABI default
        (piko_draw only enqueues; errors surface at a later draw or finish)."""
        import torch
        bin_h = bin_w if bin_h is None else bin_h
        self.device = torch.device(device or "cuda")
        with torch.cuda.device(self.device):
            self.ctx = piko_create(width, height, bin_w, bin_h)
        if sync == "checked":
            piko_set_sync(self.ctx, PIKO_SYNC_CHECKED)
        elif sync != "async":
            raise ValueError("sync must be 'checked' or 'async'")
        self.W, self.H, self.bin_w, self.bin_h = width, height, bin_w, bin_h
        self.rgba = torch.empty((height, width, 4), dtype=torch.float32, device=self.device)
        self.depth = torch.empty((height, width), dtype=torch.float32, device=self.device)

    @property
    def n_bins(self):
        return (-(-self.W // self.bin_w)) * (-(-self.H // self.bin_h))

    def draw(self, verts, idx, mvp, light, stream=None, check=True, indexed=True):
        """indexed=True passes n_verts = verts.shape[0] (piko_draw_indexed);
        False uses the north-star piko_draw (vertex count derived on device)."""
        if indexed:
            return piko_draw_indexed(self.ctx, verts, verts.shape[0], idx, idx.shape[0], mvp, light,
                                     self.rgba, self.depth, stream, check)
        return piko_draw(self.ctx, verts, idx, idx.shape[0], mvp, light, self.rgba, self.depth,
                         stream, check)

    def draw_patches(self, patches, mvp, light, dice_px=2.0, max_grid=128, stream=None, check=True):
        return piko_draw_patches(self.ctx, patches, mvp, light, dice_px, max_grid, self.rgba, self.depth,
                                 stream, check)

    def diced(self):
        """(verts f32[V][8], idx i32[T][3]) of the last draw_patches, as torch copies."""
        import torch
        v, nv, i, nt = piko_get_diced(self.ctx)
        return (_wrap_device(v, (nv, 8), torch.float32, self.device),
                _wrap_device(i, (nt, 3), torch.int32, self.device))

    def primid(self):
        import torch
        return _wrap_device(piko_get_primid(self.ctx), (self.H, self.W), torch.int32, self.device)

    def coverage(self):
        import torch
        return _wrap_device(piko_get_coverage(self.ctx), (self.H, self.W), torch.int32, self.device)

    def bins(self):
        """(bin_start i32[NB+1], bin_prims i32[P]) as torch tensors (copies)."""
        import torch
        s, q, n = piko_get_bins(self.ctx)
        start = _wrap_device(s, (self.n_bins + 1,), torch.int32, self.device)
        prims = _wrap_device(q, (n,), torch.int32, self.device) if n else torch.zeros(0, dtype=torch.int32)
        return start, prims

    def stats(self):
        return piko_get_stats(self.ctx)

    def close(self):
        if self.ctx:
            piko_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _DevView:
    """Zero-copy __cuda_array_interface__ view of a ctx-owned device buffer."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 2}


def _wrap_device(ptr, shape, dtype, device):
    """Copy a ctx-owned device buffer into a fresh torch tensor (device-to-device)."""
    import torch
    typestr = {torch.int32: "<i4", torch.float32: "<f4", torch.int64: "<i8"}[dtype]
    torch.cuda.synchronize(device)
    if int(torch.tensor(shape).prod()) == 0:
        return torch.empty(shape, dtype=dtype, device=device)
    return torch.as_tensor(_DevView(ptr, shape, typestr), device=device).clone()
