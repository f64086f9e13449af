/*
 * piko.h -- C ABI of the B200-native binned triangle rasterizer (the one
 * data-parallel hot path of Piko, arXiv 1404.6293).
 *
 * The operation (sec. 7.1 "Baseline Rasterizer": Vertex
 * Shader -> Rasterizer -> Fragment Shader -> Depth Test -> Composite, run as
 * the binned pipeline of sec. 7.2.2; shading per Listing 1,
 * P:514-545): draw an indexed triangle list with a model-view-projection
 * matrix and a directional light into a colour buffer and a depth buffer.
 * The path inside piko_draw is
 *   vertex transform + fixed-point setup      ("Vertex Shader")
 *   AssignBin: bbox -> tiles, count, exclusive scan, stable scatter into per-bin
 *              lists in primitive order       (Table 3
 *              AssignToBoundingBox; P:1081-1084 prefix sums "while maintaining
 *              primitive order")
 *   Schedule:  one CTA per bin (LoadBalance); across GPUs bin b is
 *              owned by rank b mod R (DirectMap round robin)
 *   Process:   per bin, fixed-point edge coverage, depth test with a packed
 *              64-bit (depth, primID) minimum, Lambert shade, write-back.
 * The exact result (bit-exact coverage/depth/primID/bin lists) is defined in
 * DESIGN.md ("Readings of the paper", R1..R18) and by the CPU oracle in
 * oracle/piko_oracle.c, which this library does not share code with.
 *
 * Conventions for every entry point:
 *  - Pointers marked "device" must be CUDA device memory of the device that
 *    was current when the context was created (e.g. torch CUDA tensors);
 *    pointers marked "host" are ordinary (preferably pinned) host memory.
 *  - Device input buffers must be 16-byte aligned (vectorised loads).
 *  - The caller owns every buffer it passes; the library keeps no caller
 *    pointer beyond the stream work enqueued by that call.  The context owns
 *    its scratch (setup records, pair lists, bin CSR, primID and key buffers).
 *  - Return codes: PIKO_OK (0) or a negative PIKO_E* code; piko_last_error()
 *    gives a message.  A context serves one host thread at a time.
 */
#ifndef PIKO_H_
#define PIKO_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct piko_ctx piko_ctx;

enum {
  PIKO_OK = 0,
  PIKO_EINVAL = -1,    /* invalid argument                                   */
  PIKO_ENOMEM = -2,    /* device or host allocation failed                   */
  PIKO_ECUDA = -3,     /* a CUDA call or kernel failed                       */
  PIKO_ENCCL = -4,     /* NCCL unavailable or an NCCL call failed            */
  PIKO_ECAPACITY = -5, /* pair-list capacity exceeded and could not grow     */
  PIKO_ESTATE = -6     /* call not valid in the context's current state      */
};

/* piko_set_debug flags */
#define PIKO_DEBUG_COVERAGE_COUNT 1u /* count covering triangles per pixel   */

/* piko_set_pipeline pipelines */
#define PIKO_PIPE_BINNED 0   /* default: the binned rasterizer (sec. 7.2.2)   */
#define PIKO_PIPE_FREEPIPE 1 /* FreePipe design alternative (sec. 7.2.1,
                                P:1273-1294): one fused kernel, one thread per
                                triangle, full-screen 64-bit atomicMin keys, a
                                resolve/shade pass; no bin lists, one GPU.   */
#define PIKO_PIPE_BASELINE 2 /* Baseline design alternative (sec. 7.1,
                                P:1160-1164): VS, Rasterizer,
                                Fragment Shader, Depth Test, Composite as
                                separate kernels, full-screen bins,
                                LoadBalance (thread per triangle / fragment),
                                fragment buffers in HBM between stages (grown
                                on overflow: PIKO_ECAPACITY + re-issue); no
                                bin lists, one GPU.                           */

/* piko_set_sync modes */
#define PIKO_SYNC_CHECKED 0 /* piko_draw waits for the frame, checks the pair
                               capacity, regrows and re-issues on overflow;
                               returns after the frame completed.             */
#define PIKO_SYNC_ASYNC 1   /* default: piko_draw only enqueues
                               and returns; up to 8 frames are in flight per
                               context (the 9th draw waits for the oldest).
                               A finished frame's status is read without
                               blocking at the next piko_draw: an error of an
                               earlier frame (PIKO_ECAPACITY -- that frame's
                               outputs are invalid and the capacity has grown
                               before this draw was enqueued -- or PIKO_ECUDA)
                               is returned once, by the next piko_draw or by
                               piko_finish.                                   */

/* Create a context for a width x height framebuffer binned into bin_w x bin_h
 * pixel tiles (AssignToBoundingBox bins; Listing 1 uses 8x8).
 *   1 <= width, height <= 16384 (guard band, R2);
 *   bin_w, bin_h powers of two in [8, 64].
 * Bins form a ceil(width/bin_w) x ceil(height/bin_h) row-major grid,
 * bin = ty * binsX + tx; edge bins may be partial (R13).
 * Uses the CUDA device current on the calling thread.
 * Returns NULL on error (message via piko_last_error(NULL)).                 */
piko_ctx *piko_create(int width, int height, int bin_w, int bin_h);

/* Render one frame: asynchronous on `stream` (the default PIKO_SYNC_ASYNC
 * mode returns PIKO_OK once the frame is enqueued; see piko_set_sync).
 * Multi-GPU: a rank that overflowed its pair capacity sends empty bins and a
 * status word with its keys; rank 0 then reports PIKO_ECAPACITY for the frame.
 *   verts     device, f32[n_verts][8] = {px,py,pz,pad, nx,ny,nz,pad}
 *             (object-space position and normal, R15)
 *   idx       device, i32[n_tris][3]; caller guarantees 0 <= idx < n_verts
 *   n_tris    0 <= n_tris; the primitive ID of triangle t is t
 *   mvp       host, f32[16] row-major, clip = M * (x,y,z,1); copied at call time
 *   light     host, f32[3], direction toward the light (Listing 1 lightvec,
 *             normalised inside); copied at call time
 *   out_rgba  device, f32[height][width][4], row 0 = top; background (0,0,0,0)
 *   out_depth device, f32[height][width]; window depth in [0,1], 1.0 = clear
 *   stream    a cudaStream_t (NULL = legacy default stream)
 * After piko_attach_comm with nranks > 1, only rank 0's out_* receive the frame
 * (others may pass NULL) and every rank must pass identical scene buffers.
 * Errors: PIKO_EINVAL for null pointers with n_tris > 0, n_tris < 0, misaligned
 * buffers, a non-finite or zero light; PIKO_ECAPACITY; PIKO_ECUDA.
 * n_tris == 0 clears the outputs.                                             */
int piko_draw(piko_ctx *ctx, const float *verts, const int32_t *idx, int32_t n_tris,
              const float mvp[16], const float light[3], float *out_rgba, float *out_depth,
              void *stream);

/* piko_draw with the vertex count given: 0 <= idx < n_verts (n_verts >= 1 when
 * n_tris > 0).  piko_draw, which has no vertex count, first derives
 * n_verts = max(idx) + 1 with a device reduction over idx (one extra kernel
 * reading 12 bytes per triangle); otherwise the two calls are identical.    */
int piko_draw_indexed(piko_ctx *ctx, const float *verts, int64_t n_verts, const int32_t *idx,
                      int32_t n_tris, const float mvp[16], const float light[3], float *out_rgba,
                      float *out_depth, void *stream);

/* End-to-end variant of piko_draw on HOST buffers: copies verts (n_verts x 8
 * f32) and idx to context-owned device buffers, draws, copies rgba and depth
 * back into host buffers, and synchronises `stream` before returning.
 * Host buffers should be pinned (cudaHostRegister / torch pin_memory) for
 * full PCIe bandwidth.  Same errors as piko_draw.                            */
int piko_draw_host(piko_ctx *ctx, const float *h_verts, int64_t n_verts, const int32_t *h_idx,
                   int32_t n_tris, const float mvp[16], const float light[3], float *h_rgba,
                   float *h_depth, void *stream);

/* Pipelined end-to-end variant of piko_draw_host: returns once the frame's
 * upload, draw and download are enqueued.  Two context-owned device staging
 * slots alternate: the upload of frame k+1 (on an internal copy stream) runs
 * while frame k draws on `stream` and frame k-1 downloads (on a second copy
 * stream), so a sequence of calls is bound by the slowest of H2D, draw and
 * D2H instead of their sum.  `stream` is ordered after this frame's download:
 * synchronising it (or piko_finish) completes the frame.  The host buffers
 * must stay valid, h_verts / h_idx unmodified and h_rgba / h_depth unread,
 * until then; they must be pinned (cudaHostAlloc / cudaHostRegister / torch
 * pin_memory) for the copies to be asynchronous (pageable memory still gives
 * the right frame, synchronously).  Errors of the draw are asynchronous as
 * for piko_draw in PIKO_SYNC_ASYNC mode (an overflowed frame is reported by a
 * later call or by piko_finish; its staged image is the background).       */
int piko_draw_host_async(piko_ctx *ctx, const float *h_verts, int64_t n_verts,
                         const int32_t *h_idx, int32_t n_tris, const float mvp[16],
                         const float light[3], float *h_rgba, float *h_depth, void *stream);

/* Reyes micropolygon pipeline (sec. 5
 * "Reyes": Split -> Dice -> Sample -> Shade).  Draws n_patches bicubic Bezier
 * patches: Split/Dice on the device into a micropolygon mesh (DESIGN.md
 * R19-R21: per-patch rates Gu x Gv = the smallest powers of two <= max_grid
 * with the projected control-polyline length <= dice_px * G; quads split into
 * two triangles), then the binned Sample stage (AssignBin + per-bin raster;
 * the paper uses 32x32 bins, P:1199-1201 -- create the context with 32x32) and
 * Shade, exactly as piko_draw draws the mesh.
 *   patches  device, f32[n_patches][16][4] = (x, y, z, pad); control point
 *            a*4 + b, a along u, b along v; 16-byte aligned
 *   dice_px  > 0, target micropolygon edge (screen pixels, L-inf)
 *   max_grid power of two in [1, 1024] (caps Gu, Gv)
 * Other arguments as piko_draw.  The mesh lives in the context (see
 * piko_get_diced) until the next call; the call synchronises `stream` once
 * (mesh size readback between the rate and mesh kernels).  PIKO_ESTATE after
 * piko_attach_comm or with the FreePipe/Baseline pipelines.                  */
int piko_draw_patches(piko_ctx *ctx, const float *patches, int32_t n_patches, const float mvp[16],
                      const float light[3], float dice_px, int32_t max_grid, float *out_rgba,
                      float *out_depth, void *stream);

/* The micropolygon mesh of the last piko_draw_patches (device pointers owned
 * by the context: verts f32[n_verts][8], idx i32[n_tris][3]).               */
int piko_get_diced(const piko_ctx *ctx, const float **d_verts, int64_t *n_verts,
                   const int32_t **d_idx, int64_t *n_tris);

/* Wait for every frame in flight; returns the first error of any frame not
 * yet reported (PIKO_ECAPACITY if its pair lists overflowed -- the capacity
 * has then been grown for the next frame), else PIKO_OK.                      */
int piko_finish(piko_ctx *ctx);

/* Select PIKO_SYNC_ASYNC (default) or PIKO_SYNC_CHECKED.                      */
int piko_set_sync(piko_ctx *ctx, int mode);

/* Select the pipeline (PIKO_PIPE_BINNED, _FREEPIPE or _BASELINE).  Outputs
 * are identical; FreePipe and Baseline produce no bin lists (piko_get_bins ->
 * PIKO_ESTATE) and do not support partitions or communicators (PIKO_ESTATE). */
int piko_set_pipeline(piko_ctx *ctx, int pipeline);

/* Pixel-shader complexity (the paper's design-space axis, sec. 7.2.1,
 * "As shader complexity increases, the computation time of
 * shading a primitive significantly outweighs the time spent loading the
 * primitive").  Adds `iters` dependent float FMAs per shaded fragment:
 * forward = 1 charges every covered fragment that passes the depth range,
 * inside the raster loop (binned: per-bin CTAs, LoadBalance; FreePipe: the
 * triangle's own thread, DirectMap) -- the paper's pipelines shade before the
 * depth test; forward = 0 charges once per resolved pixel (deferred).
 * The extra result never reaches the outputs (which stay bit-identical for
 * every setting); it is kept live through a never-taken store.  Single-GPU
 * pipelines only (the multi-GPU resolve ignores it).  Applies from the next
 * draw.  EINVAL unless 0 <= iters <= PIKO_MAX_SHADER_ITERS and forward is 0
 * or 1.                                                                      */
#define PIKO_MAX_SHADER_ITERS (1 << 20)
int piko_set_shader_cost(piko_ctx *ctx, int iters, int forward);

/* Destroy; NULL-safe; synchronises internal work first.                       */
void piko_destroy(piko_ctx *ctx);

/* Last error message of ctx (ctx == NULL: the calling thread's last
 * piko_create error).  Owned by the library.                                  */
const char *piko_last_error(const piko_ctx *ctx);

/* Inspection (parity tests).  Device pointers owned by ctx, valid until the
 * next draw/destroy, readable after the frame's stream work completed.
 * primID buffer: i32[height][width], -1 = background.                         */
int piko_get_primid(const piko_ctx *ctx, const int32_t **d_primid);

/* Bin lists of the last frame as CSR: bin_start i32[NB+1], bin_prims i32[P],
 * ascending primID within each bin.  Bins not owned by this
 * rank are empty.  *n_pairs = P.  Blocks until the frame completed.           */
int piko_get_bins(const piko_ctx *ctx, const int32_t **d_bin_start, const int32_t **d_bin_prims,
                  int64_t *n_pairs);

/* Debug flags (PIKO_DEBUG_COVERAGE_COUNT: u32[height][width] number of
 * triangles covering each pixel centre, counted before the depth discard).   */
int piko_set_debug(piko_ctx *ctx, unsigned flags);
int piko_get_coverage(const piko_ctx *ctx, const uint32_t **d_covcount);

/* Sort-first partition without a communicator ("virtual rank"): rasterize only
 * bins b with b mod nranks == rank and write only their pixels.  Used to test
 * the partition on one GPU.  nranks == 1 restores the full frame.            */
int piko_set_partition(piko_ctx *ctx, int rank, int nranks);

/* The two device steps of the sort-first exchange, exposed so the multi-GPU
 * data path can be exercised on one GPU (NCCL needs one device per rank).
 * piko_draw_tile_keys: with a partition set (piko_set_partition), render this
 *   rank's owned bins into packed 64-bit (depth, primID) tile keys -- exactly
 *   the payload rank r sends to rank 0 in piko_draw.
 *     d_tile_keys  device, u64[owned_max][bin_w*bin_h]; owned bin k is
 *                  b = rank + k*nranks; pixel p = ly*bin_w + lx;
 *                  0xFFFFFFFFFFFFFFFF = no fragment.  owned_max =
 *                  ceil(NB / nranks); piko_tile_keys_count gives its length.
 * piko_resolve_keys: rank 0's step after the gather: shade gathered keys
 *     d_all_keys   device, u64[nranks][owned_max][bin_w*bin_h], rank-major
 *   into out_rgba / out_depth (and the context's primID buffer).
 * Scene arguments as in piko_draw_indexed.  Both are asynchronous on stream. */
int piko_draw_tile_keys(piko_ctx *ctx, const float *verts, int64_t n_verts, const int32_t *idx,
                        int32_t n_tris, const float mvp[16], const float light[3],
                        uint64_t *d_tile_keys, void *stream);
int piko_resolve_keys(piko_ctx *ctx, const float *verts, int64_t n_verts, const int32_t *idx,
                      int32_t n_tris, const float mvp[16], const float light[3], int nranks,
                      const uint64_t *d_all_keys, float *out_rgba, float *out_depth, void *stream);
int64_t piko_tile_keys_count(const piko_ctx *ctx);

/* Host-only (no CUDA): the bins owned by `rank` of `nranks` in payload order
 * (owned bin k = rank + k*nranks, DirectMap round robin P:688) for a
 * width x height screen in bin_w x bin_h bins.  Writes min(count, cap) bin ids
 * to out_bins (may be NULL) and returns the count, or PIKO_EINVAL.          */
int64_t piko_owned_bins(int width, int height, int bin_w, int bin_h, int rank, int nranks,
                        int32_t *out_bins, int64_t cap);

/* Multi-GPU sort-first: attach an NCCL communicator built from a
 * 128-byte ncclUniqueId that the caller broadcast to all ranks (e.g. through
 * torch.distributed).  Each rank transforms all triangles, rasterizes the bins
 * it owns (b mod nranks == rank) into packed 64-bit tile keys, and the keys are
 * gathered to rank 0 with grouped ncclSend/ncclRecv; rank 0 shades and writes
 * the frame.  NCCL is loaded at run time (libnccl.so.2).                      */
int piko_attach_comm(piko_ctx *ctx, const void *nccl_unique_id, int rank, int nranks);

/* Multi-GPU decomposition used by piko_attach_comm / piko_set_partition
 * (call before them; PIKO_ESTATE once a communicator is attached).
 *   PIKO_MULTI_SORT_FIRST (default): screen partition, above.
 *   PIKO_MULTI_SORT_LAST (the "Tiled Depth-Based
 *     Composition" row of the paper's Table 1): rank r renders the
 *     triangle range [t0_r, t0_{r+1}), t0_r = floor(n_tris*r/nranks) rounded
 *     down to a multiple of 4 (t0_nranks = n_tris), over ALL bins into packed
 *     keys with global primIDs; the key images are combined on rank 0 with
 *     ncclReduce(ncclMin, ncclUint64) -- the (depth, primID) minimum is
 *     associative and commutative, so the result is bit-identical -- and rank 0
 *     shades.  With a partition (virtual rank) piko_draw_tile_keys writes that
 *     rank's full key image, u64[NB][bin_w*bin_h] (owned_max = NB), and
 *     piko_resolve_keys(nranks = 1) shades the element-wise minimum.         */
#define PIKO_MULTI_SORT_FIRST 0
#define PIKO_MULTI_SORT_LAST 1
int piko_set_multi(piko_ctx *ctx, int mode);

/* Transport of the sort-first tile exchange (call before piko_attach_comm):
 *   PIKO_XPORT_NCCL (default): k_tile writes keys locally, then grouped
 *     ncclSend/ncclRecv to rank 0, then rank 0's resolve kernel.
 *   PIKO_XPORT_P2P (SURVEY 8(e) "fused v2"): rank 0 owns the exchange buffer
 *     u64[2][nranks][owned_max][bin_w*bin_h] (double-buffered by frame parity)
 *     plus arrival flags; the other ranks map it with CUDA IPC over NVLink
 *     during piko_attach_comm.  Each rank's tile kernel stores its keys
 *     straight into rank 0's buffer as bins finish (the transfer overlaps the
 *     raster), then its last CTA raises the rank's arrival flag (system-scope
 *     release); rank 0's resolve kernel waits for all flags (acquire) and
 *     releases the slot when read.  No NCCL call per frame.  A flag wait that
 *     exceeds 10 s reports PIKO_ENCCL instead of hanging.  Sort-first only. */
#define PIKO_XPORT_NCCL 0
#define PIKO_XPORT_P2P 1
int piko_set_transport(piko_ctx *ctx, int transport);

/* The P2P transport between contexts of ONE process on one device ("virtual
 * ranks", for tests): attach rank 0 with root == ctx first, then the other
 * ranks with the rank-0 context as root; they share its buffers.  Draw ranks
 * 1..nranks-1 before rank 0 (rank 0's resolve waits for their flags), and
 * destroy rank 0 last.                                                       */
int piko_attach_local_peers(piko_ctx *ctx, piko_ctx *root, int rank, int nranks);

/* The P2P transport without a communicator, between processes (the handle
 * bytes travel by any channel, e.g. torch.distributed):
 *   rank 0:  piko_p2p_export fills PIKO_P2P_HANDLE_BYTES of CUDA IPC handles
 *            of its exchange buffers (allocated here);
 *   rank r:  piko_p2p_import maps them.
 * Afterwards piko_draw runs the P2P exchange exactly as after
 * piko_attach_comm with PIKO_XPORT_P2P (which uses these two steps with an
 * ncclBroadcast of the handles).  Destroy rank 0's context last.            */
#define PIKO_P2P_HANDLE_BYTES 128
int piko_p2p_export(piko_ctx *ctx, int nranks, void *out_handles);
int piko_p2p_import(piko_ctx *ctx, const void *handles, int rank, int nranks);

/* Host-only (no CUDA): sort-last triangle range [*t0, *t1) of `rank` of
 * `nranks` for n_tris triangles (see PIKO_MULTI_SORT_LAST).  PIKO_EINVAL on
 * bad arguments.                                                             */
int piko_triangle_range(int64_t n_tris, int rank, int nranks, int64_t *t0, int64_t *t1);

/* Frame statistics of the last frame (blocks until it completed).            */
typedef struct {
  int64_t n_tris;       /* triangles submitted                                */
  int64_t n_live;       /* triangles surviving setup culls (owned bins > 0)   */
  int64_t n_pairs;      /* (bin, triangle) pairs, P                           */
  int64_t n_bins;       /* bins in the grid, NB                               */
  int64_t owned_bins;   /* bins rasterized by this rank                        */
  int64_t pair_capacity;/* current pair-list capacity                          */
  int32_t radix_passes; /* LSD passes the radix AssignBin would take          */
  int32_t kernels_per_frame; /* kernels launched per frame (this rank)        */
  int32_t assign_mode;  /* AssignBin of the last frame: 0 stable LSD radix passes,
                           1 count matrix (k_cm_scan + k_cm_scatter),
                           2 chunk lists (sorted in k_setup + k_cl_bins)        */
  int32_t reserved;
  int64_t cm_rows;      /* count-matrix rows / chunk-list chunks (triangle
                           chunks), 0 in radix mode                            */
} piko_stats;
int piko_get_stats(const piko_ctx *ctx, piko_stats *out);

/* Fill a 128-byte ncclUniqueId (ncclGetUniqueId) for piko_attach_comm; call
 * on rank 0 and broadcast the bytes.  PIKO_ENCCL if NCCL cannot be loaded.   */
int piko_nccl_unique_id(void *out_id128);

/* Per-stage device timing with CUDA events recorded on the frame's stream
 * between the kernels of every frame (no host synchronisation is added).
 * Stages: */
#define PIKO_STAGE_CLEAR 0   /* resets (only when a grid size changed)        */
#define PIKO_STAGE_VERTEX 1  /* k_index_max (piko_draw only) + k_vertex      */
#define PIKO_STAGE_SETUP 2   /* k_setup: setup, count, scan, pairs           */
#define PIKO_STAGE_EXPAND 3  /* k_radix_pass pass 0: expand pairs + digit-0 rank
                                (+ k_bin_scan when radix_passes == 1);
                                count-matrix mode: k_cm_scan (column prefixes,
                                bin_start)                                      */
#define PIKO_STAGE_SORT 4    /* k_radix_pass passes >= 1 (+ CSR bin scan CTAs);
                                count-matrix mode: k_cm_scatter (stable scatter
                                of every row's pairs + work lists)              */
#define PIKO_STAGE_TILE 5    /* k_tile: per-bin raster, depth, shade, store   */
#define PIKO_STAGE_GATHER 6  /* tile-key gather (multi-GPU: NCCL, or nothing for P2P) */
#define PIKO_STAGE_RESOLVE 7 /* k_resolve: rank-0 shade of gathered keys      */
#define PIKO_NUM_STAGES 8
/* on != 0 enables recording and resets the totals. */
int piko_set_profiling(piko_ctx *ctx, int on);
/* Synchronises, then returns per-stage total milliseconds and frame count
 * since profiling was enabled.                                               */
int piko_get_profile(piko_ctx *ctx, double ms[PIKO_NUM_STAGES], int64_t *frames);

#ifdef __cplusplus
}
#endif
#endif /* PIKO_H_ */
