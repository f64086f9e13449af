// kernels.cu -- the hot path of the binned rasterizer, hand-written for sm_100a.
//
//   k_setup      Vertex transform + fixed-point triangle setup + AssignBin count,
//                fused with a decoupled-look-back exclusive scan of the per-
//                triangle pair counts and a cooperative, coalesced expansion of
//                the (bin, primID) pairs in primitive order, the per-bin counts
//                (warp-aggregated) and the digit histograms of the radix passes.
//                ("Vertex Shader"; P:684 AssignToBoundingBox;
//                 P:1081-1084 prefix sums "while maintaining primitive order")
//   k_radix_pass One stable LSD pass (8-bit digit) of the pairs by bin id: warp
//                match-any ranking, per-digit decoupled look-back (16 chunks per
//                probe), shared-memory staged scatter.  Pass 0 also runs the
//                exclusive scan of the per-bin counts (CSR bin_start) in extra
//                CTAs.  After the last pass the values are the CSR bin_prims,
//                ascending primID within each bin.
//   k_tile       Process, one CTA per owned bin (LoadBalance):
//                a shared-memory tile z-buffer of packed 64-bit (depth, primID)
//                keys, setup records double-buffered into shared memory with
//                cp.async, triangle-parallel raster for small triangles and
//                pixel-parallel raster for large ones, then per-pixel Lambert
//                shade (Listing 1) and a vectorised write-back.
//   k_resolve    multi-GPU rank 0: shade the gathered tile keys into the frame.
//
// Arithmetic follows DESIGN.md R1..R18 with a pinned float op order (IEEE
// round-to-nearest intrinsics, explicit fma); this TU is compiled with
// --fmad=false so no other contraction can happen.
#include <algorithm>
#include <cstddef>
#include <cstdint>

#include "piko_internal.h"

namespace piko {

typedef unsigned long long u64;

constexpr u64 CLEAR_KEY = 0xFFFFFFFFFFFFFFFFull;
constexpr float W_EPS = 1e-6f;
constexpr float GUARD = 4194304.0f;  // 2^22 subpixels

// ---------------------------------------------------------------------------
// synchronisation helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void st_release64(u64* p, u64 v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ u64 ld_acquire64(const u64* p) {
  u64 v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed64(u64* p, u64 v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ u64 ld_relaxed64(const u64* p) {
  u64 v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// system scope: flags exchanged with peer GPUs over NVLink (P2P transport)
__device__ __forceinline__ void st_release_sys64(u64* p, u64 v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ u64 ld_acquire_sys64(const u64* p) {
  u64 v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ u64 gtimer_ns();
// Spin until *p >= want (signed compare); after P2P_TIMEOUT_NS a peer is
// presumed dead: flag the frame (host reports PIKO_ENCCL) instead of hanging.
constexpr unsigned long long P2P_TIMEOUT_NS = 10ull * 1000 * 1000 * 1000;
static __device__ __noinline__ void p2p_wait_geq(const u64* p, long long want, unsigned* timeout_flag) {
  const u64 t0 = gtimer_ns();
  while ((long long)ld_acquire_sys64(p) < want) {
    __nanosleep(256);
    if (gtimer_ns() - t0 > P2P_TIMEOUT_NS) { atomicExch(timeout_flag, 1u); return; }
  }
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// optional per-CTA phase timestamps (debug builds: -DPIKO_K1_TIMING)
__device__ __forceinline__ u64 gtimer() {
  u64 t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ u64 gtimer_ns() { return gtimer(); }
#ifdef PIKO_K1_TIMING
// [kernel: 0 setup, 1 radix pass 0, 2 radix pass 1, 3 tile][slot][phase]
__device__ u64 g_k1_times[4][8192][8];
#define K1_MARK(i) do { if (threadIdx.x == 0 && chunk < 8192) g_k1_times[0][chunk][i] = gtimer(); } while (0)
#define RX_MARK(i) do { if (threadIdx.x == 0 && chunk < 8192 && a.pass < 2) g_k1_times[1 + a.pass][chunk][i] = gtimer(); } while (0)
#define TL_MARK(slot, i) do { if (threadIdx.x == 0 && (slot) < 8192) g_k1_times[3][slot][i] = gtimer(); } while (0)
__device__ __forceinline__ void g_tl_extra(int job, int n, int cta) { g_k1_times[3][job][3] = n; g_k1_times[3][job][4] = cta; }
#define TL_CTA(i) do { if (threadIdx.x == 0 && blockIdx.x < 1024) g_k1_times[0][7000 + blockIdx.x][i] = gtimer(); } while (0)
#define SCAN_MARK(tile, i) do { if (threadIdx.x == 0 && (tile) < 64 && a.pass < 2) g_k1_times[1 + a.pass][8100 + (tile)][i] = gtimer(); } while (0)
// count-matrix kernels reuse the radix slots: [1] k_cm_scan CTA j, [2] k_cm_scatter CTA
#define CM_MARK(k, slot, i) do { if (threadIdx.x == 0 && (slot) < 8000) g_k1_times[k][slot][i] = gtimer(); } while (0)
// look-back detail of radix passes 0/1 (thread 0 = digit 0): [pass][chunk]
// {level-1 end time, level-1 probes, level-2 probes, group-aggregate publish time}
__device__ u64 g_rx_lb[2][8192][8];
#define RX_LB(i, v) do { if (threadIdx.x == 0 && chunk < 8192 && a.pass < 2) g_rx_lb[a.pass][chunk][i] = (v); } while (0)
}  // namespace piko
extern "C" int piko_dbg_k1_times(void* host, size_t bytes) {
  return (int)cudaMemcpyFromSymbol(host, piko::g_k1_times, bytes);
}
extern "C" int piko_dbg_k1_set(const void* host, size_t bytes) {
  return (int)cudaMemcpyToSymbol(piko::g_k1_times, host, bytes);
}
extern "C" int piko_dbg_rx_lb(void* host, size_t bytes) {
  return (int)cudaMemcpyFromSymbol(host, piko::g_rx_lb, bytes);
}
namespace piko {
#else
#define K1_MARK(i) do { } while (0)
#define RX_MARK(i) do { } while (0)
#define RX_LB(i, v) do { } while (0)
#define TL_MARK(slot, i) do { } while (0)
#define g_tl_extra(a, b, c) do { } while (0)
#define TL_CTA(i) do { } while (0)
#define SCAN_MARK(tile, i) do { } while (0)
#define CM_MARK(k, slot, i) do { } while (0)
#endif

// Look-back status word: tag (frame+1, 20 bits) | flag (2 bits) | value (42 bits)
constexpr unsigned LB_AGG = 1u, LB_INC = 2u;
__device__ __forceinline__ u64 lb_pack(unsigned tag, unsigned flag, u64 v) {
  return ((u64)tag << 44) | ((u64)flag << 42) | v;
}
__device__ __forceinline__ unsigned lb_tag(u64 s) { return (unsigned)(s >> 44); }
__device__ __forceinline__ unsigned lb_flag(u64 s) { return (unsigned)(s >> 42) & 3u; }
__device__ __forceinline__ u64 lb_val(u64 s) { return s & ((1ull << 42) - 1); }
__device__ __forceinline__ unsigned frame_tag(u64 frame) { return (unsigned)((frame + 1) & 0xFFFFFu); }

// Decoupled look-back (one full warp): publish this chunk's aggregate, sum the
// predecessors back to the nearest inclusive prefix, 128 per probe (4 per lane,
// lane-major: entry q = hi - 32*j - lane); publish the inclusive prefix.
// Returns the exclusive prefix.
static // Status words carry their own payload (tag, flag and value in one 64-bit
// word), so relaxed atomic loads/stores suffice: an acquire load per probe
// entry would add a fence per load to the chain.
__device__ u64 lookback_warp(u64* status, long long chunk, u64 agg, unsigned tag, int lane) {
  if (lane == 0) st_relaxed64(&status[chunk], lb_pack(tag, chunk == 0 ? LB_INC : LB_AGG, agg));
  if (chunk == 0) return 0;
  u64 excl = 0;
  long long hi = chunk - 1;
  for (;;) {
    u64 sv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const long long i = hi - 32 * j - lane;
      sv[j] = (i >= 0) ? ld_relaxed64(&status[i]) : lb_pack(tag, LB_INC, 0);
    }
    // walk the 4 groups of 32 in order (nearest predecessors first)
    bool retry = false, done = false;
    u64 add = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (retry || done) continue;
      const bool ready = lb_tag(sv[j]) == tag;
      const unsigned inc = __ballot_sync(0xffffffffu, ready && lb_flag(sv[j]) == LB_INC);
      const unsigned notready = __ballot_sync(0xffffffffu, !ready);
      const int k = inc ? (__ffs(inc) - 1) : 32;
      const unsigned need = (k >= 31) ? 0xffffffffu : ((2u << k) - 1u);
      if (notready & need) { retry = true; continue; }  // unpublished predecessor
      u64 v = (lane <= k) ? lb_val(sv[j]) : 0ull;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      add += v;
      hi -= 32;
      if (k < 32) done = true;
    }
    excl += add;   // groups consumed before a retry stay consumed (hi advanced)
    if (done) break;
  }
  if (lane == 0) st_relaxed64(&status[chunk], lb_pack(tag, LB_INC, excl + agg));
  return excl;
}

// ---------------------------------------------------------------------------
// vertex transform and triangle setup (R2-R4, R7, R11)
// ---------------------------------------------------------------------------
struct Tri {
  int X0, Y0, X1, Y1, X2, Y2;
  float zw0, zw1, zw2;
  float rw0, rw1, rw2;
  int v0, v1, v2;
  long long area2;
  int px0, py0, px1, py1;
  int small;
};

// Part j (0..2) of triangle t's 48-byte setup record: interleaved (default,
// [T][3]) or in three planes ([3][stride], PIKO_REC_SOA=1: the parts of
// consecutive triangles contiguous -- fewer, fuller sectors per warp on runs
// of consecutive primIDs, yet measured slower: c3 +2, c4 +17, c5 +25 us).
#ifndef PIKO_REC_SOA
#define PIKO_REC_SOA 0
#endif
__device__ __forceinline__ long long rec_at(long long t, int j, long long stride) {
#if PIKO_REC_SOA
  return (long long)j * stride + t;
#else
  (void)stride;
  return 3 * t + j;
#endif
}

__device__ __forceinline__ bool xform_corner(const float4 p, const Mat4& M, float hw, float hh,
                                             int& X, int& Y, float& zw, float& rw) {
  const float cx = __fmaf_rn(M.m[0], p.x, __fmaf_rn(M.m[1], p.y, __fmaf_rn(M.m[2], p.z, M.m[3])));
  const float cy = __fmaf_rn(M.m[4], p.x, __fmaf_rn(M.m[5], p.y, __fmaf_rn(M.m[6], p.z, M.m[7])));
  const float cz = __fmaf_rn(M.m[8], p.x, __fmaf_rn(M.m[9], p.y, __fmaf_rn(M.m[10], p.z, M.m[11])));
  const float cw = __fmaf_rn(M.m[12], p.x, __fmaf_rn(M.m[13], p.y, __fmaf_rn(M.m[14], p.z, M.m[15])));
  if (!(isfinite(cx) && isfinite(cy) && isfinite(cz) && isfinite(cw))) return false;
  if (!(cw > W_EPS)) return false;
  // 1/w: __frcp_rn is the correctly rounded IEEE reciprocal, bit-identical to
  // the oracle's 1.0f / w (round to nearest even) without a general division
  const float r = __frcp_rn(cw);
  const float xn = __fmul_rn(cx, r), yn = __fmul_rn(cy, r), zn = __fmul_rn(cz, r);
  const float sx = __fmaf_rn(xn, hw, hw);
  const float sy = __fmaf_rn(-yn, hh, hh);            // y down, row 0 = top
  const float z01 = __fmaf_rn(zn, 0.5f, 0.5f);        // GL NDC z -> [0,1]
  const float fx = __fmul_rn(sx, 256.0f), fy = __fmul_rn(sy, 256.0f);
  if (!(fabsf(fx) <= GUARD && fabsf(fy) <= GUARD)) return false;
  X = __float2int_rn(fx);                              // ties to even
  Y = __float2int_rn(fy);
  zw = z01;
  rw = r;
  return true;
}

__device__ __forceinline__ float4 load_pos(const float* __restrict__ verts, int vid) {
  return __ldg(reinterpret_cast<const float4*>(verts + 8ll * vid));
}

// Vertex stage record (O1 output): {X, Y, bits(zw), bits(rw)} or X = VX_CULLED.
__device__ __forceinline__ int4 transform_vertex(float4 p, const Mat4& M, int W, int H) {
  const float hw = __fmul_rn(0.5f, __int2float_rn(W));
  const float hh = __fmul_rn(0.5f, __int2float_rn(H));
  int X, Y;
  float zw, rw;
  if (!xform_corner(p, M, hw, hh, X, Y, zw, rw)) return make_int4(VX_CULLED, 0, 0, 0);
  return make_int4(X, Y, __float_as_int(zw), __float_as_int(rw));
}

// Triangle setup (O2-O4) from the three transformed corners; false = culled.
__device__ __forceinline__ bool setup_tri(int4 c0, int4 c1, int4 c2, int i0, int i1, int i2, int W,
                                          int H, Tri& o) {
  if (c0.x == VX_CULLED || c1.x == VX_CULLED || c2.x == VX_CULLED) return false;
  o.X0 = c0.x; o.Y0 = c0.y; o.zw0 = __int_as_float(c0.z); o.rw0 = __int_as_float(c0.w);
  o.X1 = c1.x; o.Y1 = c1.y; o.zw1 = __int_as_float(c1.z); o.rw1 = __int_as_float(c1.w);
  o.X2 = c2.x; o.Y2 = c2.y; o.zw2 = __int_as_float(c2.z); o.rw2 = __int_as_float(c2.w);
  o.v0 = i0; o.v1 = i1; o.v2 = i2;
  long long area2 = (long long)(o.X1 - o.X0) * (long long)(o.Y2 - o.Y0) -
                    (long long)(o.Y1 - o.Y0) * (long long)(o.X2 - o.X0);
  if (area2 == 0) return false;
  if (area2 < 0) {  // orientation normalisation: swap corners 1 and 2
    int ti; float tf;
    ti = o.X1; o.X1 = o.X2; o.X2 = ti;
    ti = o.Y1; o.Y1 = o.Y2; o.Y2 = ti;
    tf = o.zw1; o.zw1 = o.zw2; o.zw2 = tf;
    tf = o.rw1; o.rw1 = o.rw2; o.rw2 = tf;
    ti = o.v1; o.v1 = o.v2; o.v2 = ti;
    area2 = -area2;
  }
  o.area2 = area2;
  const int minX = min(o.X0, min(o.X1, o.X2)), maxX = max(o.X0, max(o.X1, o.X2));
  const int minY = min(o.Y0, min(o.Y1, o.Y2)), maxY = max(o.Y0, max(o.Y1, o.Y2));
  // sample-centre rect: ceil((min-128)/256) .. floor((max-128)/256); >> floors
  int px0 = -((128 - minX) >> 8), px1 = (maxX - 128) >> 8;
  int py0 = -((128 - minY) >> 8), py1 = (maxY - 128) >> 8;
  px0 = max(px0, 0); py0 = max(py0, 0);
  px1 = min(px1, W - 1); py1 = min(py1, H - 1);
  if (px0 > px1 || py0 > py1) return false;
  o.px0 = px0; o.py0 = py0; o.px1 = px1; o.py1 = py1;
  o.small = (maxX - minX < 32768) && (maxY - minY < 32768);
  return true;
}

// number of bins b in tile rect [tx0,tx1]x[ty0,ty1] with b % R == r
static __device__ __noinline__ unsigned owned_in_rect_r(int tx0, int ty0, int tx1, int ty1, const Grid g);
__device__ __forceinline__ unsigned owned_in_rect(int tx0, int ty0, int tx1, int ty1, const Grid& g) {
  if (g.nranks == 1) return (unsigned)((tx1 - tx0 + 1) * (ty1 - ty0 + 1));
  return owned_in_rect_r(tx0, ty0, tx1, ty1, g);
}
static __device__ __noinline__ unsigned owned_in_rect_r(int tx0, int ty0, int tx1, int ty1, const Grid g) {
  unsigned n = 0;
  const int w = tx1 - tx0 + 1;
  for (int ty = ty0; ty <= ty1; ++ty) {
    const int base = ty * g.binsX + tx0;
    const int first = (g.rank - base % g.nranks + g.nranks) % g.nranks;
    if (first < w) n += (unsigned)((w - 1 - first) / g.nranks + 1);
  }
  return n;
}

// r-th owned bin of the rect, row-major (inverse of owned_in_rect's order)
static __device__ __noinline__ int owned_bin_at_r(int tx0, int ty0, int tx1, int ty1, unsigned r, const Grid g);
__device__ __forceinline__ int owned_bin_at(int tx0, int ty0, int tx1, int ty1, unsigned r, const Grid& g) {
  const int w = tx1 - tx0 + 1;
  if (g.nranks == 1) return (ty0 + (int)(r / w)) * g.binsX + tx0 + (int)(r % w);
  return owned_bin_at_r(tx0, ty0, tx1, ty1, r, g);
}
static __device__ __noinline__ int owned_bin_at_r(int tx0, int ty0, int tx1, int ty1, unsigned r, const Grid g) {
  const int w = tx1 - tx0 + 1;
  for (int ty = ty0; ty <= ty1; ++ty) {
    const int base = ty * g.binsX + tx0;
    const int first = (g.rank - base % g.nranks + g.nranks) % g.nranks;
    const unsigned n = first < w ? (unsigned)((w - 1 - first) / g.nranks + 1) : 0u;
    if (r < n) return base + first + (int)r * g.nranks;
    r -= n;
  }
  return -1;  // unreachable for r < owned_in_rect
}

#ifndef PIKO_TILE_TU  // ---- main TU only: every kernel but k_tile ----
// ---------------------------------------------------------------------------
// K0: vertex stage -- each vertex transformed and snapped exactly once
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(VX_THREADS) k_vertex(VertexArgs a) {
#ifdef PIKO_K1_TIMING
  if (threadIdx.x == 0) {  // [0][8190]: first / last CTA start (before the wait), [0][8191]: after it
    const u64 t = gtimer();
    atomicMin(&g_k1_times[0][8190][0], t);
    atomicMax(&g_k1_times[0][8190][1], t);
  }
#endif
  pdl_wait();   // the previous frame's kernels still read xv
  pdl_trigger();
#ifdef PIKO_K1_TIMING
  if (threadIdx.x == 0) atomicMin(&g_k1_times[0][8191][0], gtimer());
#endif
  long long V = a.n_verts >= 0 ? a.n_verts : (long long)a.ctl->vmax;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.ctl->vx_need = (unsigned long long)V;
    if (V > a.cap) a.ctl->vx_overflow = 1;
  }
  V = V < a.cap ? V : a.cap;
  constexpr int VPT = VX_VPT;
  for (long long v0 = (long long)blockIdx.x * VX_THREADS * VPT + threadIdx.x; v0 < V;
       v0 += (long long)gridDim.x * VX_THREADS * VPT) {
    float4 p[VPT];
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const long long v = v0 + k * VX_THREADS;
      p[k] = v < V ? load_pos(a.verts, (int)v) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const long long v = v0 + k * VX_THREADS;
      if (v < V) a.xv[v] = transform_vertex(p[k], a.M, a.W, a.H);
    }
  }
}

// n_verts for piko_draw (no vertex count in its signature): max(idx) + 1
__global__ void __launch_bounds__(256) k_index_max(const int32_t* __restrict__ idx, long long n,
                                                   Control* ctl) {
  pdl_wait();
  pdl_trigger();
  int m = -1;
  const long long n4 = n / 4;
  const int4* p = reinterpret_cast<const int4*>(idx);
#pragma unroll 4
  for (long long i = (long long)blockIdx.x * 256 + threadIdx.x; i < n4; i += (long long)gridDim.x * 256) {
    const int4 q = __ldg(p + i);
    m = max(m, max(max(q.x, q.y), max(q.z, q.w)));
  }
  for (long long i = n4 * 4 + (long long)blockIdx.x * 256 + threadIdx.x; i < n; i += (long long)gridDim.x * 256)
    m = max(m, __ldg(idx + i));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  // one global atomic per CTA (per-warp atomics on one address serialise at L2)
  __shared__ int s_m[8];
  if ((threadIdx.x & 31) == 0) s_m[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    int mm = s_m[0];
    for (int w = 1; w < 8; ++w) mm = max(mm, s_m[w]);
    if (mm >= 0) atomicMax(&ctl->vmax, (unsigned)mm + 1u);
  }
}

// ---------------------------------------------------------------------------
// K1: triangle setup (O2-O4, O6 plane) -- a streaming kernel: setup record and
// tile rect per triangle, digit histograms of the radix passes.  The pairs are
// expanded from the rects by radix pass 0 (no scan here).
// ---------------------------------------------------------------------------
constexpr int K1_BIG = 64;  // triangles with more owned bins go to the CTA-wide loop

// FUSED: no k_vertex launch; the corners are transformed here from the raw
// positions (each shared vertex is transformed once per triangle using it --
// same arithmetic, so the same bits -- and one kernel and its 16 B/vertex
// round trip through HBM/L2 disappear).
// Shared memory of k_setup (dynamic: over the 48 KB static limit): the staged
// indices, the radix digit histograms and the large-triangle list, and the
// chunk-list AssignBin's touched-bin bitmap and per-touched-bin arrays.
struct K1Smem {
  union {                             // the staged indices are consumed before the main loop
    int4 idx[K1_CHUNK * 3 / 4];
    struct {
      uint2 big[K1_CHUNK];
      unsigned hist[MAX_PASSES][RX_RADIX];
    } rx;
  } u;
  // (launches in count-matrix / radix frames allocate only the union: the small
  // carve-out leaves the L1 to the corner gathers)
  unsigned char bigg[K1_CHUNK];       // chunk-list mode: group of a listed triangle
  uint2 mrect[K1_CHUNK];              // chunk-list: rect of slot k*K1_THREADS + tid if it owns 2..K1_BIG bins
  unsigned bm[CL_MAX_NB / 32];        // chunk-list: bins touched by the chunk
  unsigned short wpre[CL_MAX_NB / 32];  // exclusive popcount prefix of bm (local digit base)
  unsigned short tb[CL_MAX_NB];       // local digit d -> bin
  unsigned mask[CL_MAX_NB];           // by local digit: bit (k*8 + warp) = that group has a pair in the bin
  unsigned cnt[CL_MAX_NB];            // by local digit: pairs of the bin in this chunk
  unsigned wsum[K1_THREADS / 32];
  unsigned U;
};
static_assert(K1_TPT * K1_THREADS / 32 <= 32, "32-triangle groups of a chunk fit one mask word");

// ---------------------------------------------------------------------------
// Chunk-list AssignBin, first half (a3 count inside k_setup).
// The chunk's triangles form 32 groups of 32 consecutive primitives (group
// k*8 + warp = triangles t0 + 32 (k*8 + warp) + lane).  Its pairs mark the
// touched bins in a bitmap; the popcount prefix turns them into dense local
// digits; the pairs then add their group bit and count per digit.  One entry
// per touched bin b: cl_ent[b][chunk] = {group mask, pairs}, bit `chunk` of
// b's chunk bitmap, cl_tot[b] += pairs.  Work is O(pairs + NB/32 + touched).
// One-bin triangles arrive warp-aggregated (bin1); multi-bin ones through the
// big list (rect + group), their pairs spread over the CTA.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned cl_digit(const K1Smem& sm, int b) {
  return sm.wpre[b >> 5] + __popc(sm.bm[b >> 5] & ((1u << (b & 31)) - 1u));
}
template <int PHASE>  // 0: mark bins in the bitmap; 1: masks and counts by digit
__device__ __forceinline__ void cl_pairs(K1Smem& sm, const int (&bin1)[K1_TPT], unsigned mflag, unsigned nbig,
                                         const Grid& g) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int k = 0; k < K1_TPT; ++k) {
    const unsigned peers = __match_any_sync(0xffffffffu, bin1[k]);
    if (bin1[k] >= 0 && lane == __ffs(peers) - 1) {
      const int b = bin1[k];
      if (PHASE == 0) atomicOr(&sm.bm[b >> 5], 1u << (b & 31));
      else {
        const unsigned d = cl_digit(sm, b);
        atomicOr(&sm.mask[d], 1u << (k * (K1_THREADS / 32) + warp));
        atomicAdd(&sm.cnt[d], (unsigned)__popc(peers));
      }
    }
  }
  // triangles owning 2..K1_BIG bins: their own thread walks the rect
#pragma unroll
  for (int k = 0; k < K1_TPT; ++k) {
    if (!(mflag >> k & 1u)) continue;
    const uint2 rr = sm.mrect[k * K1_THREADS + tid];
    const int tx0 = rr.x & 0xffff, ty0 = rr.x >> 16, tx1 = rr.y & 0xffff, ty1 = rr.y >> 16;
    for (int ty = ty0; ty <= ty1; ++ty)
      for (int tx = tx0; tx <= tx1; ++tx) {
        const int b = ty * g.binsX + tx;
        if (g.nranks > 1 && b % g.nranks != g.rank) continue;
        if (PHASE == 0) atomicOr(&sm.bm[b >> 5], 1u << (b & 31));
        else {
          const unsigned d = cl_digit(sm, b);
          atomicOr(&sm.mask[d], 1u << (k * (K1_THREADS / 32) + warp));
          atomicAdd(&sm.cnt[d], 1u);
        }
      }
  }
  // larger ones: the whole CTA walks their bins
  for (unsigned q = 0; q < nbig; ++q) {
    const uint2 rr = sm.u.rx.big[q];
    const int tx0 = rr.x & 0xffff, ty0 = rr.x >> 16, tx1 = rr.y & 0xffff, ty1 = rr.y >> 16;
    const unsigned c = owned_in_rect(tx0, ty0, tx1, ty1, g);
    for (unsigned j = tid; j < c; j += K1_THREADS) {
      const int b = owned_bin_at(tx0, ty0, tx1, ty1, j, g);
      if (PHASE == 0) atomicOr(&sm.bm[b >> 5], 1u << (b & 31));
      else {
        const unsigned d = cl_digit(sm, b);
        atomicOr(&sm.mask[d], 1u << sm.bigg[q]);
        atomicAdd(&sm.cnt[d], 1u);
      }
    }
  }
}
__device__ __forceinline__ void cl_publish(const SetupArgs& a, K1Smem& sm, const int (&bin1)[K1_TPT],
                                           unsigned mflag, unsigned nbig, long long chunk, u64 frame) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Grid& g = a.g;
  const int NBW = (g.NB + 31) >> 5;
  // (the bitmap was zeroed before the main loop; big-list pairs are marked here)
  cl_pairs<0>(sm, bin1, mflag, nbig, g);
  __syncthreads();
  // touched bins -> local digits (words: one per thread; NBW <= CL_MAX_NB/32 <= K1_THREADS)
  static_assert(CL_MAX_NB / 32 <= K1_THREADS, "one bitmap word per thread");
  const unsigned wv = tid < NBW ? sm.bm[tid] : 0u;
  const unsigned pc = __popc(wv);
  unsigned inc = pc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) sm.wsum[warp] = inc;
  __syncthreads();
  unsigned d = inc - pc;
#pragma unroll
  for (int w = 0; w < K1_THREADS / 32; ++w) d += w < warp ? sm.wsum[w] : 0u;
  if (tid < NBW) sm.wpre[tid] = (unsigned short)d;
  if (tid == K1_THREADS - 1) sm.U = d + pc;
  for (unsigned bits = wv; bits; bits &= bits - 1) {
    sm.tb[d] = (unsigned short)(tid * 32 + __ffs(bits) - 1);
    sm.mask[d] = 0u;
    sm.cnt[d] = 0u;
    ++d;
  }
  __syncthreads();
  cl_pairs<1>(sm, bin1, mflag, nbig, g);
  __syncthreads();
  // one entry per touched bin
  const unsigned U = sm.U, cbit = 1u << (chunk & 31);
  for (unsigned q = tid; q < U; q += K1_THREADS) {
    const int b = sm.tb[q];
    const unsigned c = sm.cnt[q];
    a.cl_ent[(size_t)b * a.cl_nch + chunk] = make_uint2(sm.mask[q], c);
    atomicOr(&a.cl_bm[(size_t)b * a.cl_nw + (chunk >> 5)], cbit);
    atomicAdd(&a.cl_tot[b], c);
  }
  // the grid's last CTA scans the bin totals into bin_start (no chain between
  // CTAs: each other CTA is done once its entries are published)
  __shared__ int s_last;
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    s_last = (atomicAdd(&a.ctl->cl_done, 1ull) + 1) % gridDim.x == 0;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  constexpr int BPT = CL_MAX_NB / K1_THREADS;
  static_assert(BPT % 4 == 0, "uint4 loads");
  const int NB = g.NB;
  unsigned c[BPT];
#pragma unroll
  for (int k = 0; k < BPT; k += 4) {
    const int bb = tid * BPT + k;
    if ((NB & 3) == 0 && bb + 4 <= NB) {
      const uint4 q = __ldcg(reinterpret_cast<const uint4*>(a.cl_tot + bb));
      c[k] = q.x; c[k + 1] = q.y; c[k + 2] = q.z; c[k + 3] = q.w;
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) c[k + u] = bb + u < NB ? __ldcg(a.cl_tot + bb + u) : 0u;
    }
  }
  u64 cs = 0;
#pragma unroll
  for (int k = 0; k < BPT; ++k) cs += c[k];
  u64 inc64 = cs;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u64 t = __shfl_up_sync(0xffffffffu, inc64, o);
    if (lane >= o) inc64 += t;
  }
  __shared__ u64 s_w64[K1_THREADS / 32];
  if (lane == 31) s_w64[warp] = inc64;
  __syncthreads();
  u64 run = inc64 - cs, P = 0;
#pragma unroll
  for (int w = 0; w < K1_THREADS / 32; ++w) {
    run += w < warp ? s_w64[w] : 0ull;
    P += s_w64[w];
  }
#pragma unroll
  for (int k = 0; k < BPT; ++k) {
    const int bb = tid * BPT + k;
    if (bb < NB) a.cl_start[bb] = (int32_t)(run < MAX_PAIRS ? run : MAX_PAIRS - 1);
    run += c[k];
  }
  if (tid == 0) {
    a.ctl->n_pairs = P;
    a.cl_start[NB] = (int32_t)(P < MAX_PAIRS ? P : MAX_PAIRS - 1);
    if (P > a.cl_cap) atomicMax(&a.ctl->overflow_tag, frame + 1);
  }
}

template <bool FUSED>
#ifndef PIKO_K1_MINB
#define PIKO_K1_MINB 3
#endif
__global__ void __launch_bounds__(K1_THREADS, PIKO_K1_MINB) k_setup(SetupArgs a) {
  extern __shared__ __align__(16) unsigned char k1_dyn[];
  K1Smem& sm1 = *reinterpret_cast<K1Smem*>(k1_dyn);
  unsigned (&s_hist)[MAX_PASSES][RX_RADIX] = sm1.u.rx.hist;
  uint2 (&s_big)[K1_CHUNK] = sm1.u.rx.big;
  __shared__ unsigned s_nbig;
  __shared__ u64 s_tk;
  __shared__ unsigned s_live;
  const int tid = threadIdx.x;
  const Grid g = a.g;

  // (the index loads below read only the caller's input: they are issued
  // before the dependency wait, so CTAs resident early overlap k_vertex)
  // every CTA takes one ticket per frame: frame = ticket / gridDim.x (the
  // triangle chunk is simply blockIdx.x -- nothing here depends on CTA order)
  const long long chunk = blockIdx.x;
  const long long t0 = chunk * K1_CHUNK;
  K1_MARK(0);
  // ---- the chunk's indices: 16-byte coalesced loads staged in shared memory
  // (12 consecutive ints per 4 triangles; t0 is a multiple of K1_CHUNK and idx
  // is 16-byte aligned), issued together with the frame ticket --------------
  int4 (&s_idx)[K1_CHUNK * 3 / 4] = sm1.u.idx;
  const u64 tk = a.frame * gridDim.x;  // (host frame counter: no same-address atomic burst)
  {
    const long long nint = 3 * (min((long long)K1_CHUNK, a.n_tris - t0));
    const long long n4 = nint >> 2;
    const int4* ip = reinterpret_cast<const int4*>(a.idx + 3 * t0);
    int4 q[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int j = tid + k * K1_THREADS;
      q[k] = j < n4 ? __ldg(ip + j) : make_int4(-1, -1, -1, -1);
      if (j == n4 && (nint & 3)) {  // ragged tail: 1-3 ints
        int* qi = reinterpret_cast<int*>(&q[k]);
        for (int u = 0; u < (int)(nint & 3); ++u) qi[u] = __ldg(a.idx + 3 * t0 + 4 * n4 + u);
      }
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) s_idx[tid + k * K1_THREADS] = q[k];
  }
  const bool cl = a.cl_ent != nullptr;  // chunk-list AssignBin (CTA-uniform)
  if (cl)
    for (int i = tid; i < ((g.NB + 31) >> 5); i += K1_THREADS) sm1.bm[i] = 0u;
  if (tid == 0) { s_tk = tk / gridDim.x; s_live = 0; s_nbig = 0; }
  pdl_wait();   // k_vertex output; the previous frame's kernels read rec / rect / the count matrix
  pdl_trigger();
  __syncthreads();  // indices staged; histogram cleared; frame known
  const u64 frame = s_tk;
  int vi[K1_TPT][3];
  const int* sidx = reinterpret_cast<const int*>(s_idx);
#pragma unroll
  for (int k = 0; k < K1_TPT; ++k) {
    const long long t = t0 + tid + k * K1_THREADS;
    const bool in = t < a.n_tris;
#pragma unroll
    for (int c = 0; c < 3; ++c) vi[k][c] = in ? sidx[3 * (tid + k * K1_THREADS) + c] : 0;
  }
  // the index space now holds the large-triangle list and the digit histograms
  __syncthreads();
  if (a.npass > 0) {
    for (int i = tid; i < a.npass * RX_RADIX; i += K1_THREADS) (&s_hist[0][0])[i] = 0;
    __syncthreads();
  }
  // corner loads predicated per slot only (slots past n_tris are skipped
  // below); an index past the vertex records (an overflowed frame, reported
  // and discarded) is clamped in bounds
  int4 cv[K1_TPT][3];
  if constexpr (FUSED) {
    float4 pp[K1_TPT][3];
#pragma unroll
    for (int k = 0; k < K1_TPT; ++k) {
      const bool in = t0 + tid + k * K1_THREADS < a.n_tris;
#pragma unroll
      for (int c = 0; c < 3; ++c) pp[k][c] = in ? load_pos(a.verts, vi[k][c]) : make_float4(0.f, 0.f, 0.f, 1.f);
    }
#pragma unroll
    for (int k = 0; k < K1_TPT; ++k)
#pragma unroll
      for (int c = 0; c < 3; ++c) cv[k][c] = transform_vertex(pp[k][c], a.M, g.W, g.H);
  } else {
    const unsigned vlast = (unsigned)(a.xv_cap - 1);
#pragma unroll
    for (int k = 0; k < K1_TPT; ++k) {
      const bool in = t0 + tid + k * K1_THREADS < a.n_tris;
#pragma unroll
      for (int c = 0; c < 3; ++c)
        cv[k][c] = in ? __ldg(a.xv + min((unsigned)vi[k][c], vlast)) : make_int4(VX_CULLED, 0, 0, 0);
    }
  }
  K1_MARK(1);

  // ---- setup, record + rect write (coalesced: consecutive threads, t) -------
  unsigned live = 0;
  // count-matrix mode: the CTA's triangles all lie in row t0 >> cm_shift
  // (K1_CHUNK divides the row size); one-bin triangles are warp-aggregated
  uint32_t* cmrow = a.cm ? a.cm + (size_t)(t0 >> a.cm_shift) * g.NB : nullptr;
  const int warp = tid >> 5;
  int bin1[K1_TPT];
  unsigned mflag = 0;  // chunk-list: slots whose triangle owns 2..K1_BIG bins (rect in mrect)
#pragma unroll
  for (int k = 0; k < K1_TPT; ++k) {
    bin1[k] = -1;
    const long long t = t0 + tid + k * K1_THREADS;
    if (t >= a.n_tris) continue;
    uint2 rr = make_uint2(1u, 0u);  // empty rect: tx0 = 1 > tx1 = 0
    Tri o;
    if (setup_tri(cv[k][0], cv[k][1], cv[k][2], vi[k][0], vi[k][1], vi[k][2], g.W, g.H, o)) {
      const int tx0 = o.px0 >> g.bw_log2, tx1 = o.px1 >> g.bw_log2;
      const int ty0 = o.py0 >> g.bh_log2, ty1 = o.py1 >> g.bh_log2;
      const unsigned c = owned_in_rect(tx0, ty0, tx1, ty1, g);
      if (c == 1 && (cmrow || cl)) bin1[k] = g.nranks == 1 ? ty0 * g.binsX + tx0 : owned_bin_at(tx0, ty0, tx1, ty1, 0u, g);
      else if (c > 1 && c <= (unsigned)K1_BIG && cmrow) {
        for (int ty = ty0; ty <= ty1; ++ty)
          for (int tx = tx0; tx <= tx1; ++tx) {
            const int b = ty * g.binsX + tx;
            if (g.nranks > 1 && b % g.nranks != g.rank) continue;
            atomicAdd(&cmrow[b], 1u);
          }
      }
      if (c > 0) {
        rr = make_uint2((unsigned)tx0 | ((unsigned)ty0 << 16), (unsigned)tx1 | ((unsigned)ty1 << 16));
        ++live;
        // depth plane (O6) through the snapped corners
        const float dx1 = __int2float_rn(o.X1 - o.X0), dy1 = __int2float_rn(o.Y1 - o.Y0);
        const float dx2 = __int2float_rn(o.X2 - o.X0), dy2 = __int2float_rn(o.Y2 - o.Y0);
        const float dz1 = __fsub_rn(o.zw1, o.zw0), dz2 = __fsub_rn(o.zw2, o.zw0);
        const float inv = __frcp_rn(__ll2float_rn(o.area2));
        const float za = __fmul_rn(__fmaf_rn(dz1, dy2, -__fmul_rn(dz2, dy1)), inv);
        const float zb = __fmul_rn(__fmaf_rn(dz2, dx1, -__fmul_rn(dz1, dx2)), inv);
        a.rec[rec_at(t, 0, a.rec_stride)] = make_int4(o.X0, o.Y0, o.X1, o.Y1);
        a.rec[rec_at(t, 1, a.rec_stride)] = make_int4(o.X2, o.Y2, __float_as_int(o.zw0), __float_as_int(za));
        a.rec[rec_at(t, 2, a.rec_stride)] = make_int4(__float_as_int(zb), o.px0 | (o.py0 << 16),
                                                      o.px1 | (o.py1 << 16), o.small ? REC_SMALL : 0);
        // digit histograms of the radix passes over this triangle's pairs
        if (cl && c > 1 && c <= (unsigned)K1_BIG) {  // chunk-list: walked by this thread
          sm1.mrect[k * K1_THREADS + tid] = rr;
          mflag |= 1u << k;
        } else if (a.npass == 0 && c <= (unsigned)K1_BIG) {
          // count-matrix mode: no digit histograms
        } else if (c <= (unsigned)K1_BIG) {
          for (int ty = ty0; ty <= ty1; ++ty)
            for (int tx = tx0; tx <= tx1; ++tx) {
              const int b = ty * g.binsX + tx;
              if (g.nranks > 1 && b % g.nranks != g.rank) continue;
              for (int p = 0; p < a.npass; ++p) atomicAdd(&s_hist[p][(b >> (RX_BITS * p)) & (RX_RADIX - 1)], 1u);
            }
        } else {
          const unsigned q = atomicAdd(&s_nbig, 1u);
          s_big[q] = rr;
          if (cl) sm1.bigg[q] = (unsigned char)(k * (K1_THREADS / 32) + warp);  // (tail: chunk-list launches only)
        }
      }
    }
    a.rect[t] = rr;
  }
  if (cmrow) {
#pragma unroll
    for (int k = 0; k < K1_TPT; ++k) {
      const unsigned peers = __match_any_sync(0xffffffffu, bin1[k]);
      if (bin1[k] >= 0 && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&cmrow[bin1[k]], (unsigned)__popc(peers));
    }
  }
  K1_MARK(2);
  if (live) atomicAdd(&s_live, live);
  __syncthreads();
  if (chunk == 0 && tid == 0) {
    a.ctl->frame = frame; a.ctl->tile_next = 0; a.ctl->vmax = 0;
    for (int k = 0; k < NLIST; ++k) a.ctl->list_n[k] = 0;
    a.ctl->empty_next = 0; a.ctl->eq_next = 0; a.ctl->cm_touched = 0;
    if (a.ctl->vx_overflow) { a.ctl->vx_overflow = 0; atomicMax(&a.ctl->overflow_tag, frame + 1); }
  }
  // large triangles: the whole CTA walks their bins
  const unsigned nbig = s_nbig;
  if (cl) {
    cl_publish(a, sm1, bin1, mflag, nbig, chunk, frame);
  } else {
    for (unsigned q = 0; q < nbig; ++q) {
      const uint2 rr = s_big[q];
      const int tx0 = rr.x & 0xffff, ty0 = rr.x >> 16, tx1 = rr.y & 0xffff, ty1 = rr.y >> 16;
      const unsigned c = owned_in_rect(tx0, ty0, tx1, ty1, g);
      for (unsigned j = tid; j < c; j += K1_THREADS) {
        const int b = owned_bin_at(tx0, ty0, tx1, ty1, j, g);
        for (int p = 0; p < a.npass; ++p) atomicAdd(&s_hist[p][(b >> (RX_BITS * p)) & (RX_RADIX - 1)], 1u);
        if (cmrow) atomicAdd(&cmrow[b], 1u);
      }
    }
  }
  __syncthreads();
  for (int i = tid; i < a.npass * RX_RADIX; i += K1_THREADS) {
    const unsigned v = (&s_hist[0][0])[i];
    if (v) atomicAdd(&a.ctl->digit_hist[frame & 1][0][0] + i, v);
  }
  if (tid == 0 && s_live) atomicAdd(&a.ctl->n_live[frame & 1], (u64)s_live);
  K1_MARK(5);
}

// ---------------------------------------------------------------------------
// Bin scan (run by extra CTAs of radix pass 0): bin_count -> bin_start
// ---------------------------------------------------------------------------
static __device__ __noinline__ void schedule_bins(const RadixArgs& a, long long b0, const unsigned (&c)[SCAN_ITEMS], bool active = true);
static __device__ __noinline__ void bin_scan_tile(const RadixArgs& a, long long tile, unsigned tag) {
  __shared__ unsigned s_wsum[SCAN_THREADS / 32];
  __shared__ u64 s_base;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long b0 = tile * SCAN_CHUNK + (long long)tid * SCAN_ITEMS;
  unsigned c[SCAN_ITEMS], sum = 0;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    c[k] = (b0 + k < a.NB) ? a.bin_count[b0 + k] : 0u;
    sum += c[k];
  }
  unsigned inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += v;
  }
  if (lane == 31) s_wsum[warp] = inc;
  __syncthreads();
  SCAN_MARK(tile, 2);
  unsigned wbase = 0, total = 0;
#pragma unroll
  for (int w = 0; w < SCAN_THREADS / 32; ++w) {
    const unsigned v = s_wsum[w];
    wbase += (w < warp) ? v : 0u;
    total += v;
  }
  if (warp == 0) {
    const u64 ex = lookback_warp(a.scan_status, tile, total, tag, lane);
    if (lane == 0) s_base = ex;
  }
  __syncthreads();
  SCAN_MARK(tile, 3);
  u64 run = s_base + wbase + inc - sum;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    if (b0 + k < a.NB) {
      a.bin_start[b0 + k] = (int32_t)run;
      a.bin_count[b0 + k] = 0u;  // ready for the next frame
    }
    run += c[k];
  }
  if (b0 < a.NB && b0 + SCAN_ITEMS >= a.NB) a.bin_start[a.NB] = (int32_t)run;
  schedule_bins(a, b0, c);
}

// Schedule (a6) for the SCAN_ITEMS bins b0.. of this thread with pair counts
// c[]: owned bins into k_tile's work lists (every thread of the CTA calls it).
static __device__ __noinline__ void schedule_bins(const RadixArgs& a, long long b0, const unsigned (&c)[SCAN_ITEMS], bool active) {
  const int tid = threadIdx.x, lane = tid & 31;
  // Schedule: owned bins into k_tile's work lists (the order inside a list
  // does not affect the result).  Bins with more than a.frag pairs become
  // fragments (their global key tiles are CLEAR: k_tile's last fragment resets
  // a tile after reading it).  Appends are aggregated per CTA in shared memory:
  // one global atomic per list and CTA (a chain of dependent per-warp global
  // atomics made these CTAs the last of their grid, ~16 us on c3).
  __shared__ unsigned s_ln[NLIST];
  if (tid < NLIST) s_ln[tid] = 0u;
  __syncthreads();
  const unsigned lanemask_lt = (1u << lane) - 1u;
  int kd[SCAN_ITEMS];
  unsigned loc[SCAN_ITEMS], nfk[SCAN_ITEMS];
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    const long long b = b0 + k;
    const bool own = active && b < a.NB && (a.nranks == 1 || (int)(b % a.nranks) == a.rank);
    const unsigned cnt = own ? c[k] : 0u;
    const unsigned nf = (own && cnt > (unsigned)a.frag) ? (cnt + a.frag - 1) / a.frag : 0u;
    // list 0: fragments of split bins; 1..SIZE_CLASSES: single-fragment bins by
    // size class (4 cnt > 3 frag, 2 frag, frag, else); LIST_EMPTY; -1: not owned
    const unsigned q4 = 4u * cnt;
    const int cls = q4 > 3u * (unsigned)a.frag ? 0 : q4 > 2u * (unsigned)a.frag ? 1
                  : q4 > (unsigned)a.frag ? 2 : 3;
    const int kind = !own ? -1 : (nf > 0 ? 0 : (cnt > 0 ? 1 + cls : LIST_EMPTY));
    const unsigned peers = __match_any_sync(0xffffffffu, kind);  // whole warp
    const int leader = __ffs(peers) - 1;
    unsigned l = 0;
    if (kind == 0) l = atomicAdd(&s_ln[0], nf);  // rare: variable-length append
    else if (kind > 0 && lane == leader) l = atomicAdd(&s_ln[kind], (unsigned)__popc(peers));
    const unsigned lb = __shfl_sync(0xffffffffu, l, leader);
    if (kind != 0) l = lb + __popc(peers & lanemask_lt);
    kd[k] = kind; loc[k] = l; nfk[k] = nf;
  }
  __syncthreads();
  if (tid < NLIST) {
    const unsigned n = s_ln[tid];
    s_ln[tid] = n ? atomicAdd(&a.ctl->list_n[tid], n) : 0u;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    const int b = (int)(b0 + k);
    if (kd[k] == 0) {
      for (unsigned j = 0; j < nfk[k]; ++j) a.frag_list[s_ln[0] + loc[k] + j] = make_int2(b, (int)j);
    } else if (kd[k] > 0) {
      a.bin_list[(size_t)(kd[k] - 1) * a.NB + s_ln[kd[k]] + loc[k]] = (int32_t)b;
    }
  }
}

// ---------------------------------------------------------------------------
// K3: one stable LSD radix pass over the (bin, primID) pairs.
// Pass 0 (expand) takes a chunk of triangles, expands their pairs in primitive
// order from the tile rects, counts pairs per bin, ranks by digit 0.  Later
// passes take chunks of RX_CHUNK pairs.  A chunk with more than RX_CHUNK pairs
// is ranked in sub-blocks twice (count, then scatter).
// ---------------------------------------------------------------------------
struct RadixSmem {
  unsigned short whist[RX_WARPS][RX_RADIX];  // per-warp digit counts (<= RX_CHUNK)
  unsigned keys[RX_CHUNK];
  int vals[RX_CHUNK];
  unsigned lstart[RX_RADIX];
  unsigned gstart[RX_RADIX];
  unsigned run[RX_RADIX];
  unsigned wsum[RX_WARPS];
  u64 red[RX_WARPS];
  u64 tk;
  unsigned n;
};
struct ExpandSmem {              // pass 0 only (dynamic shared memory tail)
  unsigned off[EX_MAX_TRIS];     // exclusive pair offset per triangle of the chunk
  uint2 rect[EX_MAX_TRIS];
  unsigned cnt[EX_MAX_TRIS + EX_MAX_TRIS / 32];  // owned-bin count, padded index
};
__device__ __forceinline__ int cpad(int l) { return l + (l >> 5); }

// Ranking of up to RX_CHUNK items held in registers (warp w owns items
// [w*512, w*512+512), lane-strided): per-warp digit counters in shared memory.
__device__ __forceinline__ void rank_items(const unsigned (&key)[RX_ITEMS], unsigned n, unsigned wb,
                                           int shift, unsigned short (*whist)[RX_RADIX], int warp, int lane,
                                           unsigned (&rank)[RX_ITEMS]) {
  const unsigned lanemask_lt = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < RX_ITEMS; ++j) {
    const unsigned pos = wb + j * 32;
    const bool valid = pos < n;
    const unsigned d = valid ? ((key[j] >> shift) & (RX_RADIX - 1)) : RX_RADIX;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    unsigned prev = 0;
    if (valid) prev = whist[warp][d];
    __syncwarp();
    if (valid && lane == __ffs(peers) - 1) whist[warp][d] = (unsigned short)(prev + __popc(peers));
    __syncwarp();
    rank[j] = prev + __popc(peers & lanemask_lt);
  }
}

// Expand chunk with more than RX_CHUNK pairs (triangles covering many bins):
// windows of RX_CHUNK pairs are expanded cooperatively into shared memory
// (each triangle writes the part of its pair range inside the window) and
// ranked twice -- first to count (publish), then to scatter with running
// offsets.  phase 0: count into sm.run[d] and the bin counts; phase 1: scatter
// from sm.gstart.
static __device__ __noinline__ void expand_slow(const RadixArgs& a, RadixSmem& sm, const ExpandSmem& ex,
                                         int ntri, long long t0, unsigned n, int phase) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool dig = tid < RX_RADIX;  // thread tid owns digit tid
  if (dig) {
    if (phase == 1) sm.lstart[tid] = sm.gstart[tid];
    else sm.run[tid] = 0;
  }
#pragma unroll 1
  for (unsigned lo = 0; lo < n; lo += RX_CHUNK) {
    const unsigned hi = min(n, lo + RX_CHUNK);
#pragma unroll 1
    for (int i = tid; i < RX_WARPS * RX_RADIX; i += RX_THREADS) (&sm.whist[0][0])[i] = 0;
    __syncthreads();  // previous window fully consumed
#pragma unroll 1
    for (int l = tid; l < ntri; l += RX_THREADS) {
      const unsigned c = ex.cnt[cpad(l)], o = ex.off[l];
      if (c == 0 || o >= hi || o + c <= lo) continue;
      const uint2 rr = ex.rect[l];
      const int tx0 = rr.x & 0xffff, ty0 = rr.x >> 16, tx1 = rr.y & 0xffff, ty1 = rr.y >> 16;
      const unsigned j0 = max(o, lo), j1 = min(o + c, hi);
#pragma unroll 1
      for (unsigned j = j0; j < j1; ++j) {
        sm.keys[j - lo] = (unsigned)owned_bin_at(tx0, ty0, tx1, ty1, j - o, a.g);
        sm.vals[j - lo] = (int)(t0 + l);
      }
    }
    __syncthreads();
    const unsigned m = hi - lo;
    const unsigned wb = (unsigned)warp * (RX_ITEMS * 32) + lane;
    unsigned key[RX_ITEMS], rank[RX_ITEMS];
    int val[RX_ITEMS];
#pragma unroll
    for (int j = 0; j < RX_ITEMS; ++j) {
      const unsigned pos = wb + j * 32;
      key[j] = pos < m ? sm.keys[pos] : 0u;
      val[j] = pos < m ? sm.vals[pos] : 0;
    }
    if (phase == 0) {
#pragma unroll
      for (int j = 0; j < RX_ITEMS; ++j) {  // pairs per bin (CSR), warp-aggregated
        const unsigned pos = wb + j * 32;
        const unsigned kb = pos < m ? key[j] : 0xFFFFFFFFu;
        const unsigned pb = __match_any_sync(0xffffffffu, kb);
        if (pos < m && lane == __ffs(pb) - 1) atomicAdd(&a.bin_count[kb], (unsigned)__popc(pb));
      }
    }
    rank_items(key, m, wb, a.shift, sm.whist, warp, lane, rank);
    __syncthreads();
    unsigned tot = 0;
    if (dig) {
#pragma unroll 1
      for (int w = 0; w < RX_WARPS; ++w) {
        const unsigned c = sm.whist[w][tid];
        sm.whist[w][tid] = (unsigned short)tot;
        tot += c;
      }
    }
    __syncthreads();
    if (phase == 1) {
#pragma unroll
      for (int j = 0; j < RX_ITEMS; ++j) {
        const unsigned pos = wb + j * 32;
        if (pos >= m) continue;
        const unsigned d = (key[j] >> a.shift) & (RX_RADIX - 1);
        const unsigned gpos = sm.lstart[d] + sm.whist[warp][d] + rank[j];
        if (a.keys_out) a.keys_out[gpos] = key[j];
        a.vals_out[gpos] = val[j];
      }
    }
    __syncthreads();
    if (dig) {
      if (phase == 1) sm.lstart[tid] += tot;
      else sm.run[tid] += tot;
    }
  }
  __syncthreads();
}

template <bool EXPAND>
__global__ void __launch_bounds__(RX_THREADS, RX_MIN_CTAS) k_radix_pass(RadixArgs a) {
  extern __shared__ __align__(16) unsigned char rx_smem[];
  RadixSmem& sm = *reinterpret_cast<RadixSmem*>(rx_smem);
  ExpandSmem& ex = *reinterpret_cast<ExpandSmem*>(rx_smem + sizeof(RadixSmem));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool dig = tid < RX_RADIX;  // thread tid owns digit tid (look-back, offsets)

  pdl_wait();
  pdl_trigger();
  if (tid == 0) sm.tk = atomicAdd(&a.ctl->rx_ticket[a.pass], 1ull);
  __syncthreads();
  const u64 frame = sm.tk / gridDim.x;
  const long long chunk = (long long)(sm.tk % gridDim.x);
  const unsigned tag = frame_tag(frame);

  auto block_excl = [&](unsigned v) -> unsigned {  // every thread must call it
    unsigned inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) sm.wsum[warp] = inc;
    __syncthreads();
    unsigned base = 0;
    for (int w = 0; w < warp; ++w) base += sm.wsum[w];
    __syncthreads();
    return base + inc - v;
  };
  const unsigned hist_d = dig ? a.ctl->digit_hist[frame & 1][a.pass][tid] : 0u;
  u64 P;
  bool ovf = a.ctl->overflow_tag == frame + 1;
  long long nchunks;
  if (EXPAND) {
    // P = sum of the digit-0 histogram; pass 0 checks the pair capacity
    u64 v = hist_d;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) sm.red[warp] = v;
    __syncthreads();
    P = 0;
#pragma unroll
    for (int w = 0; w < RX_WARPS; ++w) P += sm.red[w];
    if (P > a.cap) ovf = true;
    if (chunk == 0 && tid == 0) {
      a.ctl->n_pairs = P;
      if (P > a.cap) atomicMax(&a.ctl->overflow_tag, frame + 1);
    }
    nchunks = ovf ? 0 : (a.n_tris + a.tri_chunk - 1) / a.tri_chunk;
  } else {
    P = ovf ? 0ull : a.ctl->n_pairs;
    nchunks = (long long)((P + RX_CHUNK - 1) / RX_CHUNK);
  }
  if (chunk >= nchunks) {
    // extra CTAs: the CSR bin scan + work lists (counts are final: pass 0 done)
    const long long tile = chunk - nchunks;
    if (a.scan_here && tile < (a.NB + SCAN_CHUNK - 1) / SCAN_CHUNK) {
      SCAN_MARK(tile, 0);
      bin_scan_tile(a, tile, tag);
      SCAN_MARK(tile, 1);
    }
    return;
  }
  RX_MARK(0);
#pragma unroll
  for (int i = tid; i < RX_WARPS * RX_RADIX; i += RX_THREADS) (&sm.whist[0][0])[i] = 0;

  // ---- chunk contents ----------------------------------------------------------
  unsigned key[RX_ITEMS];
  int val[RX_ITEMS];
  unsigned rank[RX_ITEMS];
  unsigned n;
  long long t0 = 0;
  int ntri = 0;
  bool fast = true;
  const unsigned wb = (unsigned)warp * (RX_ITEMS * 32) + lane;
  if (!EXPAND) {
    const u64 c0 = (u64)chunk * RX_CHUNK;
    n = (unsigned)min((u64)RX_CHUNK, P - c0);
#pragma unroll
    for (int j = 0; j < RX_ITEMS; ++j) {
      const unsigned pos = wb + j * 32;
      key[j] = pos < n ? a.keys_in[c0 + pos] : 0u;
      val[j] = pos < n ? a.vals_in[c0 + pos] : 0;
    }
  } else {
    // rect -> owned-bin count per triangle (coalesced: triangle tid + 256 k),
    // exclusive scan in triangle order (thread owns tpt consecutive triangles)
    t0 = chunk * (long long)a.tri_chunk;
    ntri = (int)min((long long)a.tri_chunk, a.n_tris - t0);
    const int tpt = a.tri_chunk / RX_THREADS;
    constexpr int TPT_MAX = EX_MAX_TRIS / RX_THREADS;
    uint2 rr[TPT_MAX];
#pragma unroll
    for (int k = 0; k < TPT_MAX; ++k) {  // all loads in flight together
      const int l = tid + k * RX_THREADS;
      rr[k] = (l < ntri) ? a.rect[t0 + l] : make_uint2(1u, 0u);
    }
#pragma unroll
    for (int k = 0; k < TPT_MAX; ++k) {
      const int l = tid + k * RX_THREADS;
      if (k < tpt) {
        ex.rect[l] = rr[k];
        ex.cnt[cpad(l)] = owned_in_rect(rr[k].x & 0xffff, rr[k].x >> 16, rr[k].y & 0xffff, rr[k].y >> 16, a.g);
      }
    }
    __syncthreads();
    RX_MARK(5);
    unsigned sum = 0;
#pragma unroll 1
    for (int k = 0; k < tpt; ++k) sum += ex.cnt[cpad(tid * tpt + k)];
    unsigned run = block_excl(sum);
#pragma unroll 1
    for (int k = 0; k < tpt; ++k) {
      ex.off[tid * tpt + k] = run;
      run += ex.cnt[cpad(tid * tpt + k)];
    }
    if (tid == RX_THREADS - 1) sm.n = run;
    __syncthreads();
    n = sm.n;
    fast = n <= RX_CHUNK;
    RX_MARK(6);
    if (fast) {  // expand into shared memory, thread per triangle (coalesced order)
#pragma unroll 1
      for (int k = 0; k < tpt; ++k) {
        const int l = tid + k * RX_THREADS;
        if (l >= ntri) break;
        const unsigned c = ex.cnt[cpad(l)];
        if (c == 0) continue;
        const uint2 r2 = ex.rect[l];
        const int tx0 = r2.x & 0xffff, ty0 = r2.x >> 16, tx1 = r2.y & 0xffff, ty1 = r2.y >> 16;
        unsigned o = ex.off[l];
#pragma unroll 1
        for (int ty = ty0; ty <= ty1; ++ty)
#pragma unroll 1
          for (int tx = tx0; tx <= tx1; ++tx) {
            const int b = ty * a.g.binsX + tx;
            if (a.g.nranks > 1 && b % a.g.nranks != a.g.rank) continue;
            sm.keys[o] = (unsigned)b;
            sm.vals[o] = (int)(t0 + l);
            ++o;
          }
      }
      __syncthreads();
      RX_MARK(7);
#pragma unroll
      for (int j = 0; j < RX_ITEMS; ++j) {
        const unsigned pos = wb + j * 32;
        key[j] = pos < n ? sm.keys[pos] : 0u;
        val[j] = pos < n ? sm.vals[pos] : 0;
      }
    }
  }
  RX_MARK(1);

  // ---- per-digit chunk totals, published before the ranking ------------------
  unsigned total;
  if (fast) {
    if (dig) sm.run[tid] = 0;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < RX_ITEMS; ++j) {  // warp-aggregated: few distinct digits per chunk
      const bool valid = wb + j * 32 < n;  // (spatially coherent bins, high digits) would
      const unsigned d = valid ? ((key[j] >> a.shift) & (RX_RADIX - 1)) : RX_RADIX;  // serialise
      const unsigned peers = __match_any_sync(0xffffffffu, d);
      if (valid && lane == __ffs(peers) - 1) atomicAdd(&sm.run[d], (unsigned)__popc(peers));
    }
    __syncthreads();
    total = dig ? sm.run[tid] : 0u;
  } else {
    expand_slow(a, sm, ex, ntri, t0, n, 0);
    total = dig ? sm.run[tid] : 0u;
  }
  // two-level decoupled look-back, part 1: publish.  Chunks form groups of
  // LB_GROUP; the last chunk of a group to arrive publishes the group aggregate.
  const long long grp = chunk / LB_GROUP, g0 = grp * LB_GROUP;
  const long long gsize = min((long long)LB_GROUP, nchunks - g0);
  u64* st = a.status + (size_t)chunk * RX_RADIX + tid;
  if (dig) {
    a.ccount[(size_t)chunk * RX_RADIX + tid] = total;
    st_relaxed64(st, lb_pack(tag, chunk == 0 ? LB_INC : LB_AGG, total));
  }
  __syncthreads();
  if (tid == 0) {
    RX_LB(3, 0);
    __threadfence();
    sm.n = (atomicAdd(&a.garrive[(frame & 1) * a.gcap + grp], 1u) + 1u == (unsigned)gsize) ? 1u : 0u;
    RX_LB(4, gtimer());  // arrival counted
  }
  __syncthreads();
  if (sm.n && dig) {  // last chunk of the group to arrive: publish the group aggregate
    __threadfence();
    // all LB_GROUP loads in flight together: a runtime-bounded loop would issue
    // them one L2 round trip apart (in-order issue stalls on each add), which
    // under a saturated memory system delays the group aggregate by ~20 us
    unsigned cv[LB_GROUP];
#pragma unroll
    for (int j = 0; j < LB_GROUP; ++j)
      cv[j] = j < gsize ? __ldcg(&a.ccount[(size_t)(g0 + j) * RX_RADIX + tid]) : 0u;
    unsigned gs = 0;
#pragma unroll
    for (int j = 0; j < LB_GROUP; ++j) gs += cv[j];
    RX_LB(5, gs ? gtimer() : gtimer());
    u64* gw = a.gstatus + (size_t)grp * RX_RADIX + tid;
    const u64 cur = ld_relaxed64(gw);
    if (lb_flag(cur) != LB_INC || lb_tag(cur) != tag)
      st_relaxed64(gw, lb_pack(tag, grp == 0 ? LB_INC : LB_AGG, gs));
    RX_LB(3, gtimer());
  }
  const unsigned gprefix = block_excl(hist_d);

  // ---- rank (and, expanding, count pairs per bin) while predecessors publish --
  if (fast) {
    if (EXPAND) {
#pragma unroll
      for (int j = 0; j < RX_ITEMS; ++j) {  // pairs per bin (CSR), warp-aggregated
        const unsigned pos = wb + j * 32;
        const unsigned kb = pos < n ? key[j] : 0xFFFFFFFFu;
        const unsigned pb = __match_any_sync(0xffffffffu, kb);
        if (pos < n && lane == __ffs(pb) - 1) atomicAdd(&a.bin_count[kb], (unsigned)__popc(pb));
      }
    }
    rank_items(key, n, wb, a.shift, sm.whist, warp, lane, rank);
    __syncthreads();
    if (dig) {
      unsigned tot = 0;
#pragma unroll
      for (int w = 0; w < RX_WARPS; ++w) {  // exclusive over warps
        const unsigned c = sm.whist[w][tid];
        sm.whist[w][tid] = (unsigned short)tot;
        tot += c;
      }
    }
  }
  RX_MARK(2);

  // ---- look-back part 2: walk (thread tid owns digit tid) ---------------------
  u64 excl = 0;
  if (chunk > 0 && dig) {
    bool done = false;
    unsigned np1 = 0, np2 = 0;
    // level 1: own group, chunks chunk-1 .. g0
    long long c = chunk - 1;
    while (!done && c >= g0) {
      ++np1;
      constexpr int LPROBE = LB_GROUP / 2;  // register budget of 2 CTAs/SM
      u64 sv[LPROBE];
#pragma unroll
      for (int j = 0; j < LPROBE; ++j)
        sv[j] = (c - j >= g0) ? ld_relaxed64(a.status + (size_t)(c - j) * RX_RADIX + tid) : 0ull;
      int j = 0;
#pragma unroll
      for (int q = 0; q < LPROBE; ++q) {
        if (done || j != q || c - q < g0) continue;
        if (lb_tag(sv[q]) != tag) continue;  // not yet published: stop, re-probe
        excl += lb_val(sv[q]);
        if (lb_flag(sv[q]) == LB_INC) done = true;
        ++j;
      }
      c -= j;
      if (!done && c >= g0 && j == 0) __nanosleep(32);
    }
    RX_LB(0, gtimer());
    // level 2: previous groups
    long long gq = grp - 1;
    while (!done && gq >= 0) {
      ++np2;
      constexpr int GPROBE = 8;
      u64 sv[GPROBE];
#pragma unroll
      for (int j = 0; j < GPROBE; ++j)
        sv[j] = (gq - j >= 0) ? ld_relaxed64(a.gstatus + (size_t)(gq - j) * RX_RADIX + tid)
                              : lb_pack(tag, LB_INC, 0);
      int j = 0;
#pragma unroll
      for (int q = 0; q < GPROBE; ++q) {
        if (done || j != q) continue;
        if (lb_tag(sv[q]) != tag) continue;
        excl += lb_val(sv[q]);
        if (lb_flag(sv[q]) == LB_INC) done = true;
        ++j;
      }
      gq -= j;
      if (!done && j == 0) __nanosleep(32);
    }
    st_relaxed64(st, lb_pack(tag, LB_INC, excl + total));
    RX_LB(1, np1);
    RX_LB(2, np2);
    (void)np1; (void)np2;
  }
  if (dig) {
    if (chunk == g0 + gsize - 1)  // last chunk of its group: the group's inclusive prefix
      st_relaxed64(a.gstatus + (size_t)grp * RX_RADIX + tid, lb_pack(tag, LB_INC, excl + total));
    sm.gstart[tid] = gprefix + (unsigned)excl;
  }
  RX_MARK(3);

  // ---- phase B: scatter ----------------------------------------------------------
  if (fast) {  // stage the chunk sorted by digit in shared memory, then write out
    const unsigned lstart = block_excl(total);
    if (dig) sm.lstart[tid] = lstart;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < RX_ITEMS; ++j) {
      const unsigned pos = wb + j * 32;
      if (pos < n) {
        const unsigned d = (key[j] >> a.shift) & (RX_RADIX - 1);
        const unsigned lp = sm.lstart[d] + sm.whist[warp][d] + rank[j];
        sm.keys[lp] = key[j];
        sm.vals[lp] = val[j];
      }
    }
    __syncthreads();
    for (unsigned i = tid; i < n; i += RX_THREADS) {
      const unsigned k = sm.keys[i];
      const unsigned d = (k >> a.shift) & (RX_RADIX - 1);
      const unsigned gpos = sm.gstart[d] + (i - sm.lstart[d]);
      if (a.keys_out) a.keys_out[gpos] = k;
      a.vals_out[gpos] = sm.vals[i];
    }
  } else {
    __syncthreads();
    expand_slow(a, sm, ex, ntri, t0, n, 1);
  }
  RX_MARK(4);
}

// CSR bin scan + work lists for single-pass grids (after the expand pass)
__global__ void __launch_bounds__(SCAN_THREADS) k_bin_scan(RadixArgs a) {
  __shared__ u64 s_tk;
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0) s_tk = atomicAdd(&a.ctl->scan_ticket, 1ull);
  __syncthreads();
  const u64 frame = s_tk / gridDim.x;
  bin_scan_tile(a, (long long)(s_tk % gridDim.x), frame_tag(frame));
}

// ---------------------------------------------------------------------------
// Count-matrix AssignBin (a4 exclusive scans + a5 stable scatter, DESIGN.md
// sec. 6) for NB <= CM_MAX_NB.  k_setup has added every triangle's owned bins
// into row r = t >> cm_shift of M.  The bin lists in primitive order
// then need only
//   pos(t, b) = bin_start[b] + sum_{r' < r} M[r'][b] + #{t' < t in row r : b in t'}
// k_cm_scan forms the first two terms for every (row, bin) -- a column scan,
// plus one decoupled look-back over its CTAs for bin_start -- and
// k_cm_scatter the last term inside one CTA per row: no look-back per pair
// chunk and no second sort pass.
// ---------------------------------------------------------------------------
constexpr int CM_GROUPS = 256 / CM_COLS;  // row groups per k_cm_scan CTA
constexpr int CM_RPT = 16;                // rows per thread kept in registers
__global__ void __launch_bounds__(256) k_cm_scan(const __grid_constant__ CmArgs a) {
  __shared__ unsigned s_part[CM_GROUPS][CM_COLS];
  __shared__ int s_last;
  __shared__ u64 s_w[256 / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, col = tid % CM_COLS, grp = tid / CM_COLS;
  pdl_wait();   // k_setup's counts
  pdl_trigger();
  const long long j = blockIdx.x;
  CM_MARK(1, j, 0);
  const int NB = a.g.NB;
  const long long b = j * CM_COLS + col;
  const long long rpg = (a.rows + CM_GROUPS - 1) / CM_GROUPS;
  const long long r0 = grp * rpg, r1 = min(a.rows, r0 + rpg);
  // the column slice stays in registers between the two sweeps when it is
  // short (rows <= CM_GROUPS x CM_RPT, the usual case); otherwise re-read
  unsigned sum = 0, v[CM_RPT];
  const bool cached = rpg <= CM_RPT;
  if (b < NB) {
    for (long long r = r0; r < r1; r += CM_RPT) {  // CM_RPT loads in flight
#pragma unroll
      for (int u = 0; u < CM_RPT; ++u) v[u] = (r + u < r1) ? __ldcg(a.cm + (size_t)(r + u) * NB + b) : 0u;
#pragma unroll
      for (int u = 0; u < CM_RPT; ++u) sum += v[u];
    }
  }
  s_part[grp][col] = sum;
  __syncthreads();
  CM_MARK(1, j, 1);
  if (tid < CM_COLS) {  // exclusive over the row groups of column tid; the bin total
    unsigned run = 0;
#pragma unroll
    for (int q = 0; q < CM_GROUPS; ++q) {
      const unsigned c = s_part[q][tid];
      s_part[q][tid] = run;
      run += c;
    }
    if (j * CM_COLS + tid < NB) a.sched.bin_count[j * CM_COLS + tid] = run;
  }
  __syncthreads();
  if (b < NB) {
    // second sweep: column prefixes out (bin_start is added by the scatter),
    // counts reset to zero for the next frame
    unsigned run = s_part[grp][col];
    for (long long r = r0; r < r1; r += CM_RPT) {
      if (!cached) {
#pragma unroll
        for (int u = 0; u < CM_RPT; ++u) v[u] = (r + u < r1) ? __ldcg(a.cm + (size_t)(r + u) * NB + b) : 0u;
      }
#pragma unroll
      for (int u = 0; u < CM_RPT; ++u) {
        if (r + u >= r1) break;
        const size_t o = (size_t)(r + u) * NB + b;
        a.cp[o] = run;
        run += v[u];
        if (v[u]) a.cm[o] = 0u;
      }
    }
  }
  CM_MARK(1, j, 2);
  if (NB <= RX_CHUNK) return;  // small grids: every k_cm_scatter CTA scans the totals itself
  // the last CTA to finish scans the bin totals into bin_start (no chain
  // between CTAs: every other CTA is done after its own sweeps)
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const u64 t = atomicAdd(&a.ctl->cm_done, 1ull);
    s_last = (t + 1) % gridDim.x == 0;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  u64 carry = 0;
  // steps of 256 * BPT bins, BPT consecutive per thread (all loads of a step in flight)
  constexpr int BPT = 16;
  for (int b0 = 0; b0 < NB; b0 += 256 * BPT) {
    unsigned c[BPT];
    u64 cs = 0;
    if ((NB & 3) == 0 && b0 + tid * BPT + BPT <= NB) {  // contiguous 16-byte loads (see k_cm_scatter)
#pragma unroll
      for (int k = 0; k < BPT; k += 4) {
        const uint4 q = __ldcg(reinterpret_cast<const uint4*>(a.sched.bin_count + b0 + tid * BPT + k));
        c[k] = q.x; c[k + 1] = q.y; c[k + 2] = q.z; c[k + 3] = q.w;
      }
    } else {
#pragma unroll
      for (int k = 0; k < BPT; ++k) {
        const int bb = b0 + tid * BPT + k;
        c[k] = bb < NB ? __ldcg(a.sched.bin_count + bb) : 0u;
      }
    }
#pragma unroll
    for (int k = 0; k < BPT; ++k) cs += c[k];
    u64 inc = cs;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u64 t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    u64 base = carry, tot = 0;
#pragma unroll
    for (int w = 0; w < 256 / 32; ++w) {
      base += w < warp ? s_w[w] : 0ull;
      tot += s_w[w];
    }
    u64 run = base + inc - cs;
#pragma unroll
    for (int k = 0; k < BPT; ++k) {
      const int bb = b0 + tid * BPT + k;
      if (bb < NB) a.sched.bin_start[bb] = (int32_t)(run < MAX_PAIRS ? run : MAX_PAIRS - 1);
      run += c[k];
    }
    carry += tot;
    __syncthreads();
  }
  if (tid == 0) {
    const u64 P = carry;
    a.ctl->n_pairs = P;
    a.sched.bin_start[NB] = (int32_t)(P < MAX_PAIRS ? P : MAX_PAIRS - 1);
    if (P > a.cap) atomicMax(&a.ctl->overflow_tag, a.ctl->frame + 1);
  }
  CM_MARK(1, j, 3);
}

// Stable rank by an 8-bit digit (RX_RADIX = invalid) of the items held by
// this thread: item j of warp w, lane l is number w*ipw + 32*j + l, so
// (warp, j, lane) is the items' order; per-warp digit counters in shared memory.
template <int NI>
__device__ __forceinline__ void rank_digits(const unsigned (&d)[NI], int nj,
                                            unsigned short (*whist)[RX_RADIX], int warp, int lane,
                                            unsigned (&rank)[NI]) {
  const unsigned lanemask_lt = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < NI; ++j) {
    if (j >= nj) break;  // warp-uniform
    const bool valid = d[j] < RX_RADIX;
    const unsigned peers = __match_any_sync(0xffffffffu, d[j]);
    unsigned prev = 0;
    if (valid) prev = whist[warp][d[j]];
    __syncwarp();
    if (valid && lane == __ffs(peers) - 1) whist[warp][d[j]] = (unsigned short)(prev + __popc(peers));
    __syncwarp();
    rank[j] = prev + __popc(peers & lanemask_lt);
  }
}

constexpr int CM_THREADS = 512;                  // k_cm_scatter CTA (2 per SM: 32 warps)
constexpr int CM_WARPS = CM_THREADS / 32;
constexpr int CM_ITEMS = RX_CHUNK / CM_THREADS;  // pairs of a window per thread
struct CmSmem {
  unsigned short whist[CM_WARPS][RX_RADIX];    // per-warp digit counters
  unsigned keys[RX_CHUNK];                      // window of pairs in pair order: bin
  int vals[RX_CHUNK];                           //   ... and primID
  unsigned cur[RX_CHUNK];                       // cursors: by bin (NB <= RX_CHUNK) or by local digit
  unsigned short tb[RX_CHUNK];                  // touched bin of each local digit
  unsigned bm[CM_MAX_NB / 32];                  // bins touched by the window
  unsigned short wpre[CM_MAX_NB / 32];          // exclusive popcount prefix of bm
  unsigned dtot[RX_RADIX];
  unsigned wsum[CM_WARPS];
  unsigned n, U;
};

// One CTA per count-matrix row (plus schedule CTAs).  The row's triangles are
// processed CM_SUB at a time, held in registers in warp-major order (triangle
// l = warp*TPW + 32k + lane), so (warp, k, lane) is triangle order; their
// pairs are laid out in pair order through an exclusive scan in that order
// and ranked stably per bin through dense local digits (<= 256 per ranking
// window).  Cursors start at CP[row][b] (bin_start + earlier rows).
#ifndef PIKO_CM_EARLY_OFFSETS
#define PIKO_CM_EARLY_OFFSETS 1  // k_cm_scatter: first sub-chunk's pair offsets before the dependency wait
#endif
__global__ void __launch_bounds__(CM_THREADS, 2) k_cm_scatter(const __grid_constant__ CmArgs a) {
  extern __shared__ __align__(16) unsigned char cm_smem[];
  CmSmem& sm = *reinterpret_cast<CmSmem*>(cm_smem);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NB = a.g.NB, NBW = (NB + 31) >> 5;
  const bool sched = (long long)blockIdx.x >= a.rows;
  const bool cur_by_bin = NB <= RX_CHUNK;  // the whole cursor row lives in shared memory
  const long long row = blockIdx.x;
  const long long tbeg = row << a.cm_shift, tend = sched ? tbeg : min(a.n_tris, tbeg + (1ll << a.cm_shift));
  constexpr int TPT = CM_SUB / CM_THREADS;
  constexpr int TPW = CM_SUB / CM_WARPS;   // triangles per warp
  CM_MARK(2, blockIdx.x, 0);
  // the first sub-chunk's rects (k_setup's output) are loaded before the wait
  // on k_cm_scan
  uint2 rr[TPT];
#pragma unroll
  for (int k = 0; k < TPT; ++k) {
    const long long t = tbeg + warp * TPW + k * 32 + lane;
    rr[k] = t < tend ? __ldcg(a.rect + t) : make_uint2(1u, 0u);
  }
  // owned-bin counts of the sub-chunk's triangles and their exclusive prefix
  // in (warp, k, lane) order: for the first sub-chunk this needs only
  // k_setup's rects (complete: k_cm_scan passed its own wait before this grid
  // launched), so it runs before the wait on k_cm_scan
  unsigned off[TPT], wbase = 0, n = 0;
  auto pair_offsets = [&]() {  // CTA-uniform call (one barrier)
    unsigned wrun = 0;
#pragma unroll
    for (int k = 0; k < TPT; ++k) {
      const unsigned c = owned_in_rect(rr[k].x & 0xffff, rr[k].x >> 16, rr[k].y & 0xffff, rr[k].y >> 16, a.g);
      unsigned inc = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
      }
      off[k] = wrun + inc - c;   // within the warp; the count is off-delta
      wrun += __shfl_sync(0xffffffffu, inc, 31);
    }
    __syncthreads();  // the previous reads of wsum are done
    if (lane == 0) sm.wsum[warp] = wrun;  // warp totals (wrun is warp-uniform)
    __syncthreads();
    wbase = 0; n = 0;
#pragma unroll
    for (int w = 0; w < CM_WARPS; ++w) {
      const unsigned c = sm.wsum[w];
      wbase += (w < warp) ? c : 0u;
      n += c;
    }
  };
  if (!sched && PIKO_CM_EARLY_OFFSETS) pair_offsets();
  pdl_wait();   // k_cm_scan's column prefixes and bin totals (bin_start too when NB > RX_CHUNK)
  pdl_trigger();
  CM_MARK(2, blockIdx.x, 1);
  uint32_t* cprow = a.cp + (size_t)(sched ? 0 : row) * NB;
  if (cur_by_bin) {
    // NB <= RX_CHUNK: every CTA scans the bin totals itself (BPT consecutive
    // bins per thread) -- bin_start without a serial last-CTA phase -- and
    // the cursors are bin_start + the row's column prefix, by bin
    constexpr int BPT = RX_CHUNK / CM_THREADS;
    static_assert(BPT % 4 == 0, "uint4 loads");
    unsigned c[BPT], cv[BPT];
    u64 csum = 0;
    if ((NB & 3) == 0 && tid * BPT + BPT <= NB) {
      // BPT consecutive words per thread as 16-byte loads: a warp reads one
      // contiguous run (scalar loads at this stride fetch every sector BPT times)
#pragma unroll
      for (int k = 0; k < BPT; k += 4) {
        const uint4 q = __ldcg(reinterpret_cast<const uint4*>(a.sched.bin_count + tid * BPT + k));
        c[k] = q.x; c[k + 1] = q.y; c[k + 2] = q.z; c[k + 3] = q.w;
        const uint4 r = sched ? make_uint4(0u, 0u, 0u, 0u) : __ldcg(reinterpret_cast<const uint4*>(cprow + tid * BPT + k));
        cv[k] = r.x; cv[k + 1] = r.y; cv[k + 2] = r.z; cv[k + 3] = r.w;
      }
    } else {
#pragma unroll
      for (int k = 0; k < BPT; ++k) {
        const int bb = tid * BPT + k;
        c[k] = bb < NB ? __ldcg(a.sched.bin_count + bb) : 0u;
        cv[k] = (bb < NB && !sched) ? __ldcg(cprow + bb) : 0u;
      }
    }
#pragma unroll
    for (int k = 0; k < BPT; ++k) csum += c[k];
    u64 inc = csum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u64 t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    __shared__ u64 s_w64[CM_WARPS];
    __shared__ u64 s_P;
    if (lane == 31) s_w64[warp] = inc;
    __syncthreads();
    u64 base = 0, P = 0;
#pragma unroll
    for (int w = 0; w < CM_WARPS; ++w) {
      base += w < warp ? s_w64[w] : 0ull;
      P += s_w64[w];
    }
    u64 run = base + inc - csum;
#pragma unroll
    for (int k = 0; k < BPT; ++k) {
      const int bb = tid * BPT + k;
      if (bb < NB) {
        sm.cur[bb] = (unsigned)run + cv[k];
        if (sched) a.sched.bin_start[bb] = (int32_t)(run < MAX_PAIRS ? run : MAX_PAIRS - 1);
      }
      run += c[k];
    }
    if (tid == 0) s_P = P;
    __syncthreads();
    P = s_P;
    if (sched && blockIdx.x == a.rows && tid == 0) {  // the first schedule CTA publishes P
      a.ctl->n_pairs = P;
      a.sched.bin_start[NB] = (int32_t)(P < MAX_PAIRS ? P : MAX_PAIRS - 1);
      if (P > a.cap) atomicMax(&a.ctl->overflow_tag, a.ctl->frame + 1);
    }
    if (P > a.cap) return;  // every CTA sees it: nothing is written, k_tile renders background
  }
  if (sched) {  // extra CTAs: k_tile's work lists
    const long long b0 = ((long long)blockIdx.x - a.rows) * SCAN_CHUNK + (long long)tid * SCAN_ITEMS;
    const bool active = tid < SCAN_THREADS;  // SCAN_CHUNK bins per schedule CTA
    unsigned c[SCAN_ITEMS];
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k)
      c[k] = (active && b0 + k < NB) ? __ldcg(a.sched.bin_count + b0 + k) : 0u;
    schedule_bins(a.sched, b0, c, active);
    return;
  }
  if (a.ctl->overflow_tag == a.ctl->frame + 1) return;  // P > capacity (or vertex overflow): background
  for (int w = tid; w < NBW; w += CM_THREADS) sm.bm[w] = 0u;
  auto block_excl = [&](unsigned v) -> unsigned {  // every thread must call it
    unsigned inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) sm.wsum[warp] = inc;
    __syncthreads();
    unsigned base = 0;
    for (int w = 0; w < warp; ++w) base += sm.wsum[w];
    __syncthreads();
    return base + inc - v;
  };
  for (long long sub = tbeg; sub < tend; sub += CM_SUB) {
    const bool last_sub = sub + CM_SUB >= tend;
    if (sub != tbeg) {
#pragma unroll
      for (int k = 0; k < TPT; ++k) {
        const long long t = sub + warp * TPW + k * 32 + lane;
        rr[k] = t < tend ? __ldcg(a.rect + t) : make_uint2(1u, 0u);
      }
    }
    if (sub != tbeg || !PIKO_CM_EARLY_OFFSETS) pair_offsets();
    CM_MARK(2, blockIdx.x, 3);
    for (unsigned lo = 0; lo < n; lo += RX_CHUNK) {
      const unsigned m = min((unsigned)RX_CHUNK, n - lo);
      const bool last_round = last_sub && lo + RX_CHUNK >= n;
      // expand this thread's triangles' pairs inside the window [lo, lo + m)
      // into shared memory at their pair positions
#pragma unroll
      for (int k = 0; k < TPT; ++k) {
        const int tx0 = rr[k].x & 0xffff, ty0 = rr[k].x >> 16, tx1 = rr[k].y & 0xffff, ty1 = rr[k].y >> 16;
        if (tx0 > tx1 || ty0 > ty1) continue;
        const unsigned o = wbase + off[k];
        const int val = (int)(sub + warp * TPW + k * 32 + lane);
        if (a.g.nranks == 1) {  // row-major walk of the rect part inside the window
          const int w = tx1 - tx0 + 1;
          const unsigned c = (unsigned)(w * (ty1 - ty0 + 1));
          const unsigned j0 = max(o, lo), j1 = min(o + c, lo + m);
          if (j0 >= j1) continue;
          int ty = ty0, tx = tx0;
          if (j0 > o) { ty += (int)((j0 - o) / w); tx += (int)((j0 - o) % w); }
          for (unsigned q = j0; q < j1; ++q) {
            const int b = ty * a.g.binsX + tx;
            sm.keys[q - lo] = (unsigned)b;
            sm.vals[q - lo] = val;
            if (++tx > tx1) { tx = tx0; ++ty; }
          }
        } else {
          const unsigned c = owned_in_rect(tx0, ty0, tx1, ty1, a.g);
          const unsigned j0 = max(o, lo), j1 = min(o + c, lo + m);
          for (unsigned q = j0; q < j1; ++q) {
            const int b = owned_bin_at(tx0, ty0, tx1, ty1, q - o, a.g);
            sm.keys[q - lo] = (unsigned)b;
            sm.vals[q - lo] = val;
          }
        }
      }
      __syncthreads();
      // the window's items, spread evenly over the warps (warp w holds pairs
      // [w*ipw, w*ipw + ipw)); touched-bin bitmap from the heads of runs of
      // equal bins (consecutive pairs of a coherent mesh share their bin: one
      // shared-memory atomic per run instead of a 32-way conflict per pair)
      const int ipw = (int)((m + CM_WARPS * 32 - 1) / (CM_WARPS * 32)) * 32;
      const int nj = ipw / 32;
      unsigned kb[CM_ITEMS];
#pragma unroll
      for (int j = 0; j < CM_ITEMS; ++j) {
        const unsigned pos = (unsigned)warp * ipw + j * 32 + lane;
        kb[j] = (j < nj && pos < m) ? sm.keys[pos] : 0xFFFFFFFFu;
        const unsigned prev = __shfl_up_sync(0xffffffffu, kb[j], 1);
        if (kb[j] != 0xFFFFFFFFu && (lane == 0 || prev != kb[j])) atomicOr(&sm.bm[kb[j] >> 5], 1u << (kb[j] & 31));
      }
      __syncthreads();
      if (lo == 0) CM_MARK(2, blockIdx.x, 4);
      // touched bins -> dense local digits: popcount prefix of the bitmap
      constexpr int WPT = CM_MAX_NB / 32 / CM_THREADS;  // bitmap words per thread
      unsigned wc[WPT], ws = 0;
#pragma unroll
      for (int k = 0; k < WPT; ++k) {
        const int w = tid * WPT + k;
        wc[k] = w < NBW ? sm.bm[w] : 0u;
        ws += __popc(wc[k]);
      }
      unsigned drun = block_excl(ws);
      if (tid == CM_THREADS - 1) sm.U = drun + ws;
#pragma unroll
      for (int k = 0; k < WPT; ++k) {
        const int w = tid * WPT + k;
        if (w < NBW) sm.wpre[w] = (unsigned short)drun;
        unsigned bits = wc[k];
        while (bits) {
          const int bit = __ffs(bits) - 1;
          bits &= bits - 1;
          sm.tb[drun++] = (unsigned short)(w * 32 + bit);
        }
      }
      __syncthreads();
      const unsigned U = sm.U;
      if (threadIdx.x == 0) atomicAdd(&a.ctl->cm_touched, (u64)U);
#ifdef PIKO_K1_TIMING
      if (threadIdx.x == 0 && lo == 0 && blockIdx.x < 8000) g_k1_times[2][blockIdx.x][7] = U;
#endif
      if (!cur_by_bin)
        for (unsigned d = tid; d < U; d += CM_THREADS)
          sm.cur[d] = __ldcg(cprow + sm.tb[d]) + (unsigned)__ldcg(a.sched.bin_start + sm.tb[d]);
      unsigned ld[CM_ITEMS];
      int val[CM_ITEMS];
#pragma unroll
      for (int j = 0; j < CM_ITEMS; ++j) {
        const unsigned pos = (unsigned)warp * ipw + j * 32 + lane;
        ld[j] = 0xFFFFFFFFu;
        val[j] = 0;
        if (kb[j] != 0xFFFFFFFFu) {
          val[j] = sm.vals[pos];
          ld[j] = sm.wpre[kb[j] >> 5] + __popc(sm.bm[kb[j] >> 5] & ((1u << (kb[j] & 31)) - 1u));
        }
      }
      __syncthreads();  // window and bitmap consumed (cursors loaded)
      if (lo == 0) CM_MARK(2, blockIdx.x, 5);
      for (int w = tid; w < NBW; w += CM_THREADS) sm.bm[w] = 0u;  // for the next window
      for (unsigned w0 = 0; w0 < U; w0 += RX_RADIX) {  // ranking windows of 256 local digits
        for (int i = tid; i < CM_WARPS * RX_RADIX; i += CM_THREADS) (&sm.whist[0][0])[i] = 0;
        __syncthreads();
        unsigned d[CM_ITEMS], rank[CM_ITEMS];
#pragma unroll
        for (int j = 0; j < CM_ITEMS; ++j) d[j] = (ld[j] >= w0 && ld[j] < w0 + RX_RADIX) ? ld[j] - w0 : RX_RADIX;
        rank_digits(d, nj, sm.whist, warp, lane, rank);
        __syncthreads();
        if (tid < RX_RADIX) {  // exclusive over warps (thread tid owns local digit w0 + tid)
          unsigned tot = 0;
#pragma unroll
          for (int w = 0; w < CM_WARPS; ++w) {
            const unsigned c = sm.whist[w][tid];
            sm.whist[w][tid] = (unsigned short)tot;
            tot += c;
          }
          sm.dtot[tid] = tot;
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < CM_ITEMS; ++j)
          if (j < nj && d[j] < RX_RADIX) {
            const unsigned cu = cur_by_bin ? sm.cur[sm.tb[w0 + d[j]]] : sm.cur[w0 + d[j]];
            a.bin_prims[cu + sm.whist[warp][d[j]] + rank[j]] = val[j];
          }
        __syncthreads();
        if (tid < RX_RADIX && w0 + tid < U) {
          if (cur_by_bin) sm.cur[sm.tb[w0 + tid]] += sm.dtot[tid];
          else sm.cur[w0 + tid] += sm.dtot[tid];
        }
      }
      if (lo == 0) CM_MARK(2, blockIdx.x, 6);
      if (!cur_by_bin && !last_round) {  // row cursors of the bins this row touches again
        __syncthreads();
        for (unsigned q = tid; q < U; q += CM_THREADS)
          cprow[sm.tb[q]] = sm.cur[q] - (unsigned)__ldcg(a.sched.bin_start + sm.tb[q]);
      }
      __syncthreads();
    }
  }
  CM_MARK(2, blockIdx.x, 2);
}

// ---------------------------------------------------------------------------
// Chunk-list AssignBin, second half (a4 bin scan + a5 stable scatter + a6
// schedule).  Persistent CTAs; CTA j owns bins j + k*grid.
// Every CTA scans the NB totals (bin_start of its bins, P).  For a non-empty
// bin: its chunk bitmap lists its chunks in ascending order and each chunk's
// entry {group mask, pairs} its 32-triangle groups in ascending order --
// primitive order.  Entry destinations are the exclusive scan of
// the entries' pairs; pass A loads every group's 32 rects (several per warp in
// flight) and ballots "rect holds b"; pass B (a warp per entry) walks the
// entry's groups in order and writes the primIDs.  A bin over CLB_ENT chunks
// or CLB_GRP groups flags the frame (the host falls back to the count matrix).
// CTAs past the gather part build k_tile's work lists.
// ---------------------------------------------------------------------------
struct ClbSmem {
  unsigned ch[CLB_ENT];          // entry q: chunk
  uint2 ent[CLB_ENT];            // entry q: {group mask, first group index}
  unsigned dst[CLB_ENT];         // entry q: exclusive pair offset in the bin
  unsigned grp[CLB_GRP];         // group j: global group index (triangles 32 grp + lane)
  unsigned bal[CLB_GRP];         // ballot of group j ("rect holds the bin")
  unsigned bs[CLB_KMAX], bc[CLB_KMAX];  // this CTA's bins: start, count
  u64 w64[CLB_THREADS / 32];
  unsigned ne, ng;
};
__device__ __forceinline__ u64 clb_scan64(u64 v, u64* w64, u64& tot) {  // block exclusive scan
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  u64 inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u64 t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  __syncthreads();  // (w64 may still be read by an earlier scan)
  if (lane == 31) w64[warp] = inc;
  __syncthreads();
  u64 base = 0;
  tot = 0;
#pragma unroll
  for (int w = 0; w < CLB_THREADS / 32; ++w) {
    const u64 c = w64[w];
    base += w < warp ? c : 0ull;
    tot += c;
  }
  return base + inc - v;
}

__global__ void __launch_bounds__(CLB_THREADS) k_cl_bins(const __grid_constant__ ClArgs a) {
  extern __shared__ __align__(16) unsigned char clb_dyn[];
  ClbSmem& sm = *reinterpret_cast<ClbSmem*>(clb_dyn);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NWARP = CLB_THREADS / 32;
  const int NB = a.g.NB;
  const unsigned par = (unsigned)(a.frame & 1);
  const uint32_t* tot = a.cl_tot + (size_t)par * NB;
  pdl_wait();   // k_setup's entries, bitmaps, totals and rects
  pdl_trigger();
  const bool sched = (int)blockIdx.x >= a.nbin_ctas;
  const int G = a.nbin_ctas;
  // bin_start (and P, the overflow tag) come from k_setup's last CTA
  const bool ovf = a.ctl->overflow_tag == a.frame + 1;
  if (sched) {  // k_tile's work lists (only when the frame fits)
    if (ovf) return;  // (CTA-uniform)
    const long long b0 = ((long long)blockIdx.x - a.nbin_ctas) * SCAN_CHUNK + (long long)tid * SCAN_ITEMS;
    const bool active = tid < SCAN_THREADS;
    unsigned cc[SCAN_ITEMS];
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) cc[k] = (active && b0 + k < NB) ? __ldcg(tot + b0 + k) : 0u;
    schedule_bins(a.sched, b0, cc, active);
    return;
  }
  // this CTA's bins: start and count; the other parity of the totals (read by
  // the previous frame's scan) is zeroed for the next frame's k_setup
  if (tid < CLB_KMAX) {
    const long long b = blockIdx.x + (long long)tid * G;
    if (b < NB) {
      const int s0 = __ldcg(a.sched.bin_start + b), s1 = __ldcg(a.sched.bin_start + b + 1);
      sm.bs[tid] = (unsigned)s0;
      sm.bc[tid] = (unsigned)(s1 - s0);
      a.cl_tot[(size_t)(par ^ 1u) * NB + b] = 0u;
    }
  }
  __syncthreads();
  const int wpt = (a.nw + CLB_THREADS - 1) / CLB_THREADS;
  for (int kk = 0; (long long)blockIdx.x + (long long)kk * G < NB; ++kk) {
    if (sm.bc[kk] == 0) continue;  // no entries, no bitmap bits (CTA-uniform)
    const long long b = blockIdx.x + (long long)kk * G;
    const unsigned bstart = sm.bs[kk];
    const int bx = (int)(b % a.g.binsX), by = (int)(b / a.g.binsX);
    // ---- the bin's chunks: bitmap words (thread tid holds words tid*wpt ..), zeroed
    uint32_t* bm = a.cl_bm + (size_t)b * a.nw;
    unsigned wd[CL_WPT], pc = 0;
#pragma unroll
    for (int i = 0; i < CL_WPT; ++i) {
      const int w = tid * wpt + i;
      wd[i] = (i < wpt && w < a.nw) ? __ldcg(bm + w) : 0u;
      pc += __popc(wd[i]);
    }
#pragma unroll
    for (int i = 0; i < CL_WPT; ++i)
      if (wd[i]) bm[tid * wpt + i] = 0u;
    u64 nev;
    unsigned e = (unsigned)clb_scan64(pc, sm.w64, nev);
    const unsigned ne = (unsigned)nev;
    if (ovf || ne > (unsigned)CLB_ENT) {  // (CTA-uniform)
      if (!ovf && tid == 0) { a.ctl->cl_overflow = 1u; atomicMax(&a.ctl->overflow_tag, a.frame + 1); }
      continue;
    }
#pragma unroll
    for (int i = 0; i < CL_WPT; ++i)
      for (unsigned bits = wd[i]; bits; bits &= bits - 1) sm.ch[e++] = (unsigned)((tid * wpt + i) * 32 + __ffs(bits) - 1);
    __syncthreads();
    // ---- entries {mask, pairs}: exclusive scans of pairs (destinations) and
    // groups (packed: pairs << 32 | groups), EPT consecutive entries per thread
    constexpr int EPT = CLB_ENT / CLB_THREADS;
    uint2 en[EPT];
    u64 es = 0;
#pragma unroll
    for (int u = 0; u < EPT; ++u) {
      const unsigned q = tid * EPT + u;
      en[u] = q < ne ? __ldcg(a.cl_ent + (size_t)b * a.nch + sm.ch[q]) : make_uint2(0u, 0u);
      es += ((u64)en[u].y << 32) | (unsigned)__popc(en[u].x);
    }
    u64 esum;
    u64 eo = clb_scan64(es, sm.w64, esum);
    const unsigned ng = (unsigned)esum;
    if (ng > (unsigned)CLB_GRP) {
      if (tid == 0) { a.ctl->cl_overflow = 1u; atomicMax(&a.ctl->overflow_tag, a.frame + 1); }
      continue;
    }
#pragma unroll
    for (int u = 0; u < EPT; ++u) {
      const unsigned q = tid * EPT + u;
      if (q < ne) {
        unsigned g0 = (unsigned)eo;
        sm.ent[q] = make_uint2(en[u].x, g0);
        sm.dst[q] = (unsigned)(eo >> 32);
        const unsigned gbase = sm.ch[q] * 32u;
        for (unsigned bits = en[u].x; bits; bits &= bits - 1) sm.grp[g0++] = gbase + (unsigned)(__ffs(bits) - 1);
      }
      eo += ((u64)en[u].y << 32) | (unsigned)__popc(en[u].x);
    }
    __syncthreads();
    // ---- pass A: ballots "rect holds b", 8 groups per warp in flight
    for (unsigned j0 = warp; j0 < ng; j0 += 8 * NWARP) {
      uint2 rr[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const unsigned j = j0 + u * NWARP;
        const long long t = j < ng ? (long long)sm.grp[j] * 32 + lane : a.n_tris;
        rr[u] = t < a.n_tris ? __ldcg(a.rect + t) : make_uint2(1u, 0u);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const unsigned j = j0 + u * NWARP;
        const int tx0 = rr[u].x & 0xffff, ty0 = rr[u].x >> 16, tx1 = rr[u].y & 0xffff, ty1 = rr[u].y >> 16;
        const unsigned bal = __ballot_sync(0xffffffffu, tx0 <= bx && bx <= tx1 && ty0 <= by && by <= ty1);
        if (j < ng && lane == 0) sm.bal[j] = bal;
      }
    }
    __syncthreads();
    // ---- pass B: a warp per entry walks its groups in order
    const unsigned lt = (1u << lane) - 1u;
    int32_t* out = a.bin_prims + bstart;
    for (unsigned q = warp; q < ne; q += NWARP) {
      const uint2 eq = sm.ent[q];
      unsigned o = sm.dst[q];
      const unsigned ngq = __popc(eq.x);
      for (unsigned j = eq.y; j < eq.y + ngq; ++j) {
        const unsigned bal = sm.bal[j];
        if (bal >> lane & 1u) out[o + __popc(bal & lt)] = (int32_t)(sm.grp[j] * 32u + lane);
        o += __popc(bal);
      }
    }
    __syncthreads();  // shared arrays are reused by the next bin
  }
}

// ---------------------------------------------------------------------------
// Reyes Split + Dice (R19-R21).
// k_dice_rate: one CTA; each thread decides the split/dice rate (Gu, Gv) of
// patches from their projected control hull, then a block scan over the
// patches gives every patch its first vertex and first triangle (primitive
// order = patch order, then quad (i, j), then half).  k_dice: one CTA per
// patch evaluates its (Gu+1)(Gv+1) vertices (position + Pv x Pu normal) and
// writes its 2 Gu Gv triangles.  Same pinned op order as the oracle.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int pow2_rate(float len, float dice_px, int max_grid) {
  int g = 1;
  while (g < max_grid && len > __fmul_rn(dice_px, (float)g)) g *= 2;
  return g;
}
__device__ int2 dice_rate(const float* __restrict__ cp, const Mat4& M, int W, int H, float dice_px,
                          int max_grid) {
  const float hw = __fmul_rn(0.5f, (float)W), hh = __fmul_rn(0.5f, (float)H);
  float sx[16], sy[16];
  for (int k = 0; k < 16; ++k) {
    const float x = cp[4 * k], y = cp[4 * k + 1], z = cp[4 * k + 2];
    const float cx = __fmaf_rn(M.m[0], x, __fmaf_rn(M.m[1], y, __fmaf_rn(M.m[2], z, M.m[3])));
    const float cy = __fmaf_rn(M.m[4], x, __fmaf_rn(M.m[5], y, __fmaf_rn(M.m[6], z, M.m[7])));
    const float cw = __fmaf_rn(M.m[12], x, __fmaf_rn(M.m[13], y, __fmaf_rn(M.m[14], z, M.m[15])));
    if (!(isfinite(cx) && isfinite(cy) && isfinite(cw)) || !(cw > W_EPS)) return make_int2(max_grid, max_grid);
    const float r = __frcp_rn(cw);
    sx[k] = __fmaf_rn(__fmul_rn(cx, r), hw, hw);
    sy[k] = __fmaf_rn(-__fmul_rn(cy, r), hh, hh);
  }
  float Lu = 0.0f, Lv = 0.0f;
  for (int b = 0; b < 4; ++b) {  // control rows along u: points a*4+b
    float l = 0.0f;
    for (int a = 0; a < 3; ++a) {
      const float dx = fabsf(__fsub_rn(sx[4 * (a + 1) + b], sx[4 * a + b]));
      const float dy = fabsf(__fsub_rn(sy[4 * (a + 1) + b], sy[4 * a + b]));
      l = __fadd_rn(l, dx > dy ? dx : dy);
    }
    if (l > Lu) Lu = l;
  }
  for (int a = 0; a < 4; ++a) {  // control rows along v: points a*4+b
    float l = 0.0f;
    for (int b = 0; b < 3; ++b) {
      const float dx = fabsf(__fsub_rn(sx[4 * a + b + 1], sx[4 * a + b]));
      const float dy = fabsf(__fsub_rn(sy[4 * a + b + 1], sy[4 * a + b]));
      l = __fadd_rn(l, dx > dy ? dx : dy);
    }
    if (l > Lv) Lv = l;
  }
  return make_int2(pow2_rate(Lu, dice_px, max_grid), pow2_rate(Lv, dice_px, max_grid));
}

__global__ void __launch_bounds__(1024) k_dice_rate(const __grid_constant__ DiceArgs a) {
  __shared__ unsigned long long s_w[2][32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned long long carry_v = 0, carry_t = 0;
  for (long long p0 = 0; p0 < a.n; p0 += 1024) {
    const long long p = p0 + tid;
    unsigned long long nv = 0, nt = 0;
    if (p < a.n) {
      const int2 g = dice_rate(a.patches + 64 * p, a.M, a.W, a.H, a.dice_px, a.max_grid);
      a.rate[p] = g;
      nv = (unsigned long long)(g.x + 1) * (g.y + 1);
      nt = 2ull * g.x * g.y;
    }
    unsigned long long iv = nv, it = nt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long tv = __shfl_up_sync(0xffffffffu, iv, o), tt = __shfl_up_sync(0xffffffffu, it, o);
      if (lane >= o) { iv += tv; it += tt; }
    }
    if (lane == 31) { s_w[0][warp] = iv; s_w[1][warp] = it; }
    __syncthreads();
    unsigned long long bv = carry_v, bt = carry_t, sv = 0, st = 0;
    for (int w = 0; w < 32; ++w) {
      if (w < warp) { bv += s_w[0][w]; bt += s_w[1][w]; }
      sv += s_w[0][w];
      st += s_w[1][w];
    }
    if (p < a.n) {
      a.base[2 * p] = (long long)(bv + iv - nv);
      a.base[2 * p + 1] = (long long)(bt + it - nt);
    }
    carry_v += sv;
    carry_t += st;
    __syncthreads();
  }
  if (tid == 0) { a.total[0] = (long long)carry_v; a.total[1] = (long long)carry_t; }
}

__device__ __forceinline__ void bernstein(float u, float B[4], float dB[4]) {
  const float s = __fsub_rn(1.0f, u);
  B[0] = __fmul_rn(__fmul_rn(s, s), s);
  B[1] = __fmul_rn(__fmul_rn(__fmul_rn(3.0f, u), s), s);
  B[2] = __fmul_rn(__fmul_rn(__fmul_rn(3.0f, u), u), s);
  B[3] = __fmul_rn(__fmul_rn(u, u), u);
  dB[0] = -__fmul_rn(__fmul_rn(3.0f, s), s);
  dB[1] = __fmul_rn(__fmul_rn(3.0f, s), __fsub_rn(s, __fmul_rn(2.0f, u)));
  dB[2] = __fmul_rn(__fmul_rn(3.0f, u), __fsub_rn(__fmul_rn(2.0f, s), u));
  dB[3] = __fmul_rn(__fmul_rn(3.0f, u), u);
}
__device__ __forceinline__ float comb4(const float w[4], float p0, float p1, float p2, float p3) {
  return __fmaf_rn(w[3], p3, __fmaf_rn(w[2], p2, __fmaf_rn(w[1], p1, __fmul_rn(w[0], p0))));
}

__global__ void __launch_bounds__(256) k_dice(const __grid_constant__ DiceArgs a) {
  __shared__ float s_cp[64];
  const long long p = blockIdx.x;
  if (threadIdx.x < 64) s_cp[threadIdx.x] = a.patches[64 * p + threadIdx.x];
  __syncthreads();
  const int2 g = a.rate[p];
  const int gu = g.x, gv = g.y;
  const long long vb = a.base[2 * p], tb = a.base[2 * p + 1];
  const int nvv = (gu + 1) * (gv + 1);
  for (int k = threadIdx.x; k < nvv; k += blockDim.x) {
    const int i = k / (gv + 1), j = k - i * (gv + 1);
    float Bu[4], dBu[4], Bv[4], dBv[4];
    bernstein(__fdiv_rn((float)i, (float)gu), Bu, dBu);
    bernstein(__fdiv_rn((float)j, (float)gv), Bv, dBv);
    float P[3], Pu[3], Pv[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      float Q[4], QV[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const float* row = s_cp + 16 * r + c;  // control points r*4 + 0..3, component c
        Q[r] = comb4(Bv, row[0], row[4], row[8], row[12]);
        QV[r] = comb4(dBv, row[0], row[4], row[8], row[12]);
      }
      P[c] = comb4(Bu, Q[0], Q[1], Q[2], Q[3]);
      Pu[c] = comb4(dBu, Q[0], Q[1], Q[2], Q[3]);
      Pv[c] = comb4(Bu, QV[0], QV[1], QV[2], QV[3]);
    }
    float4* v = reinterpret_cast<float4*>(a.verts + 8 * (vb + k));
    v[0] = make_float4(P[0], P[1], P[2], 0.0f);
    v[1] = make_float4(__fmaf_rn(Pv[1], Pu[2], -__fmul_rn(Pv[2], Pu[1])),
                       __fmaf_rn(Pv[2], Pu[0], -__fmul_rn(Pv[0], Pu[2])),
                       __fmaf_rn(Pv[0], Pu[1], -__fmul_rn(Pv[1], Pu[0])), 0.0f);
  }
  const int nq = gu * gv;
  for (int q = threadIdx.x; q < nq; q += blockDim.x) {
    const int i = q / gv, j = q - i * gv;
    const int v00 = (int)(vb + (long long)i * (gv + 1) + j), v01 = v00 + 1;
    const int v10 = v00 + (gv + 1), v11 = v10 + 1;
    int32_t* t = a.idx + 3 * (tb + 2ll * q);
    t[0] = v00; t[1] = v10; t[2] = v11;
    t[3] = v00; t[4] = v11; t[5] = v01;
  }
}

#endif  // PIKO_TILE_TU
// ---------------------------------------------------------------------------
// K6: per-bin Process -- raster + depth test + shade + write-back
// ---------------------------------------------------------------------------
struct RecView {
  int X0, Y0, X1, Y1, X2, Y2;
  float zw0, za, zb;
  int px0, py0, px1, py1;
  int small;
};
__device__ __forceinline__ RecView unpack(int4 q0, int4 q1, int4 q2) {
  RecView r;
  r.X0 = q0.x; r.Y0 = q0.y; r.X1 = q0.z; r.Y1 = q0.w;
  r.X2 = q1.x; r.Y2 = q1.y; r.zw0 = __int_as_float(q1.z); r.za = __int_as_float(q1.w);
  r.zb = __int_as_float(q2.x);
  r.px0 = q2.y & 0xffff; r.py0 = (unsigned)q2.y >> 16;
  r.px1 = q2.z & 0xffff; r.py1 = (unsigned)q2.z >> 16;
  r.small = q2.w & REC_SMALL;
  return r;
}

// top-left rule as a threshold: inside iff E > thr, thr = TL ? -1 : 0 (R1)
__device__ __forceinline__ int tl_thr(int Xa, int Ya, int Xb, int Yb) {
  return ((Yb == Ya && Xb > Xa) || (Yb < Ya)) ? -1 : 0;
}

// Coverage + depth at sample (Px, Py) (must lie inside the triangle's sample
// bbox when r.small).  Returns the packed key or CLEAR_KEY.
__device__ __forceinline__ u64 eval_key(const RecView& r, int Px, int Py, int t, bool& covered) {
  bool in;
  if (r.small) {
    const int e01 = (r.X1 - r.X0) * (Py - r.Y0) - (r.Y1 - r.Y0) * (Px - r.X0);
    const int e12 = (r.X2 - r.X1) * (Py - r.Y1) - (r.Y2 - r.Y1) * (Px - r.X1);
    const int e20 = (r.X0 - r.X2) * (Py - r.Y2) - (r.Y0 - r.Y2) * (Px - r.X2);
    in = e01 > tl_thr(r.X0, r.Y0, r.X1, r.Y1) && e12 > tl_thr(r.X1, r.Y1, r.X2, r.Y2) &&
         e20 > tl_thr(r.X2, r.Y2, r.X0, r.Y0);
  } else {
    const long long e01 = (long long)(r.X1 - r.X0) * (Py - r.Y0) - (long long)(r.Y1 - r.Y0) * (Px - r.X0);
    const long long e12 = (long long)(r.X2 - r.X1) * (Py - r.Y1) - (long long)(r.Y2 - r.Y1) * (Px - r.X1);
    const long long e20 = (long long)(r.X0 - r.X2) * (Py - r.Y2) - (long long)(r.Y0 - r.Y2) * (Px - r.X2);
    in = e01 > tl_thr(r.X0, r.Y0, r.X1, r.Y1) && e12 > tl_thr(r.X1, r.Y1, r.X2, r.Y2) &&
         e20 > tl_thr(r.X2, r.Y2, r.X0, r.Y0);
  }
  covered = in;
  if (!in) return CLEAR_KEY;
  const float z = __fmaf_rn(r.za, __int2float_rn(Px - r.X0),
                            __fmaf_rn(r.zb, __int2float_rn(Py - r.Y0), r.zw0));
  if (!(z >= 0.0f && z <= 1.0f)) return CLEAR_KEY;
  return ((u64)(__float_as_uint(z) & 0x7FFFFFFFu) << 32) | (unsigned)t;
}

// Prepared form of the same test (one setup per triangle, ~15 instructions per
// sample): E_ab(P) = K_ab + B_ab*dy - A_ab*dx with dx = Px - X0, dy = Py - Y0,
// A_ab = Yb - Ya, B_ab = Xb - Xa, K_ab = A_ab*(Xa - X0) - B_ab*(Ya - Y0) -- an
// exact integer identity.  For small triangles (bbox extent < 2^15) the true
// E at any sample inside the bbox fits int32, so the sum is formed modulo 2^32
// (unsigned) and is exact; large triangles use int64.
struct TriEval {
  int X0, Y0;
  int A0, B0, A1, B1, A2, B2;
  long long K1, K2;            // K01 = 0
  int thr0, thr1, thr2;        // -1 on top/left edges (R1), else 0
  float zw0, za, zb;
  int small;
};
__device__ __forceinline__ TriEval prepare(const RecView& r) {
  TriEval e;
  e.X0 = r.X0; e.Y0 = r.Y0;
  e.A0 = r.Y1 - r.Y0; e.B0 = r.X1 - r.X0;
  e.A1 = r.Y2 - r.Y1; e.B1 = r.X2 - r.X1;
  e.A2 = r.Y0 - r.Y2; e.B2 = r.X0 - r.X2;
  e.K1 = (long long)e.A1 * (r.X1 - r.X0) - (long long)e.B1 * (r.Y1 - r.Y0);
  e.K2 = (long long)e.A2 * (r.X2 - r.X0) - (long long)e.B2 * (r.Y2 - r.Y0);
  e.thr0 = tl_thr(r.X0, r.Y0, r.X1, r.Y1);
  e.thr1 = tl_thr(r.X1, r.Y1, r.X2, r.Y2);
  e.thr2 = tl_thr(r.X2, r.Y2, r.X0, r.Y0);
  e.zw0 = r.zw0; e.za = r.za; e.zb = r.zb;
  e.small = r.small;
  return e;
}
__device__ __forceinline__ u64 eval_pre(const TriEval& e, int Px, int Py, int t, bool& covered) {
  const int dx = Px - e.X0, dy = Py - e.Y0;
  bool in;
  if (e.small) {
    const unsigned udx = (unsigned)dx, udy = (unsigned)dy;
    const int E0 = (int)((unsigned)e.B0 * udy - (unsigned)e.A0 * udx);
    const int E1 = (int)((unsigned)e.K1 + (unsigned)e.B1 * udy - (unsigned)e.A1 * udx);
    const int E2 = (int)((unsigned)e.K2 + (unsigned)e.B2 * udy - (unsigned)e.A2 * udx);
    in = E0 > e.thr0 && E1 > e.thr1 && E2 > e.thr2;
  } else {
    const long long E0 = (long long)e.B0 * dy - (long long)e.A0 * dx;
    const long long E1 = e.K1 + (long long)e.B1 * dy - (long long)e.A1 * dx;
    const long long E2 = e.K2 + (long long)e.B2 * dy - (long long)e.A2 * dx;
    in = E0 > e.thr0 && E1 > e.thr1 && E2 > e.thr2;
  }
  covered = in;
  if (!in) return CLEAR_KEY;
  const float z = __fmaf_rn(e.za, __int2float_rn(dx), __fmaf_rn(e.zb, __int2float_rn(dy), e.zw0));
  if (!(z >= 0.0f && z <= 1.0f)) return CLEAR_KEY;
  return ((u64)(__float_as_uint(z) & 0x7FFFFFFFu) << 32) | (unsigned)t;
}

// O7 shade arithmetic of pixel sample (Px, Py) given triangle t's transformed
// corners (vertex-stage records) and the normals of its vertices i0..i2.
__device__ __forceinline__ float4 shade_math(int4 c0, int4 c1, int4 c2, float4 m0, float4 m1, float4 m2,
                                             int i0, int i1, int i2, int W, int H, const float L[3],
                                             int Px, int Py) {
  Tri o;
  setup_tri(c0, c1, c2, i0, i1, i2, W, H, o);      // live: t won a pixel
  const bool swapped = o.X1 != c1.x || o.Y1 != c1.y;  // O2 swapped corners 1 and 2?
  const float4 n0 = m0;
  const float4 n1 = swapped ? m2 : m1;
  const float4 n2 = swapped ? m1 : m2;
  const long long w0 = (long long)(o.X2 - o.X1) * (Py - o.Y1) - (long long)(o.Y2 - o.Y1) * (Px - o.X1);
  const long long w1 = (long long)(o.X0 - o.X2) * (Py - o.Y2) - (long long)(o.Y0 - o.Y2) * (Px - o.X2);
  const long long w2 = (long long)(o.X1 - o.X0) * (Py - o.Y0) - (long long)(o.Y1 - o.Y0) * (Px - o.X0);
  const float inv = __frcp_rn(__ll2float_rn(o.area2));
  const float l0 = __fmul_rn(__fmul_rn(__ll2float_rn(w0), inv), o.rw0);
  const float l1 = __fmul_rn(__fmul_rn(__ll2float_rn(w1), inv), o.rw1);
  const float l2 = __fmul_rn(__fmul_rn(__ll2float_rn(w2), inv), o.rw2);
  const float vx = __fmaf_rn(l2, n2.x, __fmaf_rn(l1, n1.x, __fmul_rn(l0, n0.x)));
  const float vy = __fmaf_rn(l2, n2.y, __fmaf_rn(l1, n1.y, __fmul_rn(l0, n0.y)));
  const float vz = __fmaf_rn(l2, n2.z, __fmaf_rn(l1, n1.z, __fmul_rn(l0, n0.z)));
  const float d2 = __fmaf_rn(vx, vx, __fmaf_rn(vy, vy, __fmul_rn(vz, vz)));
  float lam = 0.0f;
  if (d2 != 0.0f) {
    const float q = __fdiv_rn(__fmaf_rn(vx, L[0], __fmaf_rn(vy, L[1], __fmul_rn(vz, L[2]))),
                              __fsqrt_rn(d2));
    lam = (q > 0.0f) ? q : 0.0f;
  }
  return make_float4(__fmul_rn(0.80f, lam), __fmul_rn(0.75f, lam), __fmul_rn(0.65f, lam), 1.0f);
}

// O7 shade of pixel sample (Px, Py) by triangle t (recomputes O2 from the
// vertex-stage records; normals from the caller's vertex buffer).
static __device__ __noinline__ float4 shade(const float* __restrict__ verts, const int4* __restrict__ xv,
                                        const Mat4* M, const int32_t* __restrict__ idx, int W, int H,
                                        const float L[3], int t, int Px, int Py) {
  const int i0 = __ldg(idx + 3ll * t), i1 = __ldg(idx + 3ll * t + 1), i2 = __ldg(idx + 3ll * t + 2);
  int4 c0, c1, c2;
  if (xv) {
    c0 = __ldg(xv + i0); c1 = __ldg(xv + i1); c2 = __ldg(xv + i2);
  } else {  // fused vertex stage: the same O1 transform, recomputed
    const float4 p0 = load_pos(verts, i0), p1 = load_pos(verts, i1), p2 = load_pos(verts, i2);
    c0 = transform_vertex(p0, *M, W, H);
    c1 = transform_vertex(p1, *M, W, H);
    c2 = transform_vertex(p2, *M, W, H);
  }
  const float4 m0 = __ldg(reinterpret_cast<const float4*>(verts + 8ll * i0 + 4));
  const float4 m1 = __ldg(reinterpret_cast<const float4*>(verts + 8ll * i1 + 4));
  const float4 m2 = __ldg(reinterpret_cast<const float4*>(verts + 8ll * i2 + 4));
  return shade_math(c0, c1, c2, m0, m1, m2, i0, i1, i2, W, H, L, Px, Py);
}

// Deferred shade of N pixels of one row with every load of the dependent
// chain key -> idx -> vertex records / normals issued for all N at once
// (one chain of round trips per N pixels instead of per pixel).
template <int N>
__device__ __forceinline__ void shade_batch(const float* __restrict__ verts, const int4* __restrict__ xv,
                                            const Mat4& M, const int32_t* __restrict__ idx, int W, int H,
                                            const float L[3], const int (&t)[N], const int (&Px)[N], int Py,
                                            float4 (&c)[N]) {
  int vi[N][3];
#pragma unroll
  for (int k = 0; k < N; ++k)
#pragma unroll
    for (int j = 0; j < 3; ++j) vi[k][j] = t[k] >= 0 ? __ldg(idx + 3ll * t[k] + j) : 0;
  int4 cv[N][3];
  float4 nm[N][3];
#pragma unroll
  for (int k = 0; k < N; ++k)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      if (t[k] < 0) continue;
      if (xv) cv[k][j] = __ldg(xv + vi[k][j]);
      else {
        const float4 p = load_pos(verts, vi[k][j]);
        cv[k][j] = make_int4(__float_as_int(p.x), __float_as_int(p.y), __float_as_int(p.z), __float_as_int(p.w));
      }
      nm[k][j] = __ldg(reinterpret_cast<const float4*>(verts + 8ll * vi[k][j] + 4));
    }
#pragma unroll
  for (int k = 0; k < N; ++k) {
    c[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (t[k] < 0) continue;
    if (!xv)
#pragma unroll
      for (int j = 0; j < 3; ++j)
        cv[k][j] = transform_vertex(make_float4(__int_as_float(cv[k][j].x), __int_as_float(cv[k][j].y),
                                                __int_as_float(cv[k][j].z), __int_as_float(cv[k][j].w)), M, W, H);
    c[k] = shade_math(cv[k][0], cv[k][1], cv[k][2], nm[k][0], nm[k][1], nm[k][2], vi[k][0], vi[k][1],
                      vi[k][2], W, H, L, Px[k], Py);
  }
}

__device__ __forceinline__ void normalise_light(const float in[3], float L[3]) {
  const float s = __fsqrt_rn(__fmaf_rn(in[0], in[0], __fmaf_rn(in[1], in[1], __fmul_rn(in[2], in[2]))));
  L[0] = __fdiv_rn(in[0], s);
  L[1] = __fdiv_rn(in[1], s);
  L[2] = __fdiv_rn(in[2], s);
}

#ifndef PIKO_TINY_AREA
#define PIKO_TINY_AREA 4
#endif
constexpr int TINY_AREA = PIKO_TINY_AREA;  // clipped rect area a thread rasterizes alone
#ifndef PIKO_TINY32
#define PIKO_TINY32 1  // tiny small triangles: incremental 32-bit edge functions (0: eval_pre)
#endif
#ifndef PIKO_QSEG
#define PIKO_QSEG 4
#endif
constexpr int QSEG = PIKO_QSEG; // queued triangles: pixels of a row per work item (amortises
                                // the item search and the evaluator loads)
#ifndef PIKO_NSTAGE
#define PIKO_NSTAGE 2
#endif
constexpr int NSTAGE = PIKO_NSTAGE;  // setup-record pipeline depth (rounds in flight per warp)
constexpr int TQ = NSTAGE + 2;  // primIDs are fetched two rounds before their records

// Queue of larger triangles of the current bin (structure of arrays of the
// prepared evaluator + clipped rect), rasterized at the end of the bin by all
// threads over the flattened (triangle, pixel) index space.
template <int Q>
struct BigQueue {
  int X0[Q], Y0[Q], A0[Q], B0[Q], A1[Q], B1[Q], A2[Q], B2[Q];
  long long K1[Q], K2[Q];
  int thr[Q];                    // thr0 | thr1 << 1 | thr2 << 2 (bit set: -1), small << 3
  float zw0[Q], za[Q], zb[Q], invw[Q];
  int t[Q], rx0[Q], ry0[Q], w[Q];
  unsigned pre[Q + 1];           // exclusive prefix of the clipped areas
};

template <int BW, int BH, int THREADS>
struct TileSmem {
  static constexpr int NPX = BW * BH;
#ifndef PIKO_BIGQ_DIV
#define PIKO_BIGQ_DIV 1
#endif
#ifdef PIKO_BIGQ
  static constexpr int BIGQ = PIKO_BIGQ < THREADS ? PIKO_BIGQ : THREADS;
#else
  static constexpr int BIGQ = THREADS / PIKO_BIGQ_DIV;  // queued per bin (overflow: spill region, then warp-cooperative)
#endif
  u64 key[NPX];
  int4 rec[NSTAGE][THREADS][3];
  BigQueue<BIGQ> q;
};

// Stand-in for a longer pixel shader (ShaderCost): `iters` dependent FMAs that
// keep x in [0, 1] for x in [0, 1] (x -> x * (1 - 2^-10) + 2^-10).
__device__ __forceinline__ float shader_work(int iters, float x) {
#pragma unroll 1
  for (int i = 0; i < iters; ++i) x = __fmaf_rn(x, 0.9990234375f, 0.0009765625f);
  return x;
}
__device__ __forceinline__ float key_depth(u64 key) { return __uint_as_float((unsigned)(key >> 32)); }
__device__ __forceinline__ void shader_sink(const ShaderCost& sc, float v) {
  if (v < 0.0f) *sc.sink = v;  // unreachable: keeps the work observable
}

// Write one pixel of the frame (or the keys-only tile) from its resolved key.
template <bool COV, bool KEYS_ONLY>
__device__ __forceinline__ void store_pixel(const TileArgs& a, const float L[3], int job, int p,
                                            int npx, int x, int y, u64 key, unsigned cov) {
  if (KEYS_ONLY) {  // sort-last ranks render a triangle range: global primIDs
    a.tile_keys[(size_t)job * npx + p] = key == CLEAR_KEY ? key : key + a.prim_base;
    return;
  }
  const size_t o = (size_t)y * a.g.W + x;
  float4 c = make_float4(0.f, 0.f, 0.f, 0.f);
  float depth = 1.0f;
  int prim = -1;
  if (key != CLEAR_KEY) {
    prim = (int)(unsigned)(key & 0xFFFFFFFFu);
    depth = __uint_as_float((unsigned)(key >> 32));
#ifndef PIKO_EXP_NOSHADE
    c = shade(a.verts, a.xv, &a.M, a.idx, a.g.W, a.g.H, L, prim, 256 * x + 128, 256 * y + 128);
    if (a.sc.iters && !a.sc.forward) shader_sink(a.sc, shader_work(a.sc.iters, depth));
#endif
  }
  reinterpret_cast<float4*>(a.out_rgba)[o] = c;
  a.out_depth[o] = depth;
  a.out_primid[o] = prim;
  if (COV) a.out_cov[o] = cov;
}

template <int BW, int BH, int THREADS, bool COV, bool KEYS_ONLY>
#ifndef PIKO_EARLY_ITEM2
#define PIKO_EARLY_ITEM2 0  // 1: k_tile looks the second static item up with the first (no gain)
#endif
#ifndef PIKO_TILE_TPSM
#define PIKO_TILE_TPSM 768  // k_tile threads resident per SM the register budget is sized for
#endif
__global__ void __launch_bounds__(THREADS, PIKO_TILE_TPSM / THREADS) k_tile(const __grid_constant__ TileArgs a) {
  constexpr int NPX = BW * BH;
  constexpr int PPT = (NPX + THREADS - 1) / THREADS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TileSmem<BW, BH, THREADS>& sm = *reinterpret_cast<TileSmem<BW, BH, THREADS>*>(smem_raw);
  unsigned* s_cov = reinterpret_cast<unsigned*>(smem_raw + sizeof(TileSmem<BW, BH, THREADS>));
  __shared__ int s_bin;     // current bin (-1: work list exhausted)
  __shared__ int s_rng[5];  // its CSR sub-range [s, e), fragment count (0: whole bin), first fragment slot, fragment index
  __shared__ int s_nbig;    // large triangles queued for the pixel-parallel pass
  __shared__ unsigned s_ln[NLIST];
  __shared__ int s_last;
  __shared__ int s_nx[3];   // the next item's bin and CSR sub-range (prologue issued early)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Grid g = a.g;
  float L[3];
  normalise_light(a.light, L);
  const int fwd = a.sc.forward ? a.sc.iters : 0;  // forward shader cost per fragment
  float facc = 0.0f;
  TL_CTA(3);  // resident
  // ---- bins without pairs: background.  One ticket queue over all bins
  // (EMPTY_TICKET bins per CTA ticket, a warp takes EMPTY_TICKET/warps of
  // them); a bin is written iff it is owned and its pair count is 0.  With
  // early_empty the CTAs resident before the dependency wait already drain it:
  // the counts are final (k_cm_scan, two launches back, completed before the
  // scatter passed its own wait and triggered this launch), the empty bins are
  // never touched by the pair items, and the previous frame's k_tile is
  // complete -- so the background overlaps the scatter instead of trailing
  // the heavy bins.
  constexpr int EB_WARP = 4;                        // bins per warp per ticket
  constexpr int EMPTY_TICKET = EB_WARP * (THREADS / 32);
  __shared__ unsigned s_etk;
  auto empty_pass = [&]() {
    for (;;) {
      if (tid == 0) s_etk = atomicAdd(&a.ctl->eq_next, 1u);
      __syncthreads();
      const long long b0 = (long long)s_etk * EMPTY_TICKET + warp * EB_WARP;
      const bool done = (long long)s_etk * EMPTY_TICKET >= g.NB;
      __syncthreads();
      if (done) break;
      const long long bl = b0 + (lane & (EB_WARP - 1));
      const bool mine = lane < EB_WARP && bl < g.NB && (g.nranks == 1 || (int)(bl % g.nranks) == g.rank) &&
                        __ldcg(a.bin_count + bl) == 0u;
      const unsigned em = __ballot_sync(0xffffffffu, mine);
      for (unsigned m = em; m; m &= m - 1) {
        const int b = (int)(b0 + __ffs(m) - 1);
        const int x0 = (b % g.binsX) * BW, y0 = (b / g.binsX) * BH;
        const int x1 = min(x0 + BW, g.W) - 1, y1 = min(y0 + BH, g.H) - 1;
        const int job = (b - g.rank) / g.nranks;
        for (int p = lane; p < NPX; p += 32) {
          const int x = x0 + (p % BW), y = y0 + (p / BW);
          if (!KEYS_ONLY && (x > x1 || y > y1)) continue;
          store_pixel<COV, KEYS_ONLY>(a, L, job, p, NPX, x, y, CLEAR_KEY, 0u);
        }
      }
    }
  };
  if (a.early_empty) empty_pass();
  pdl_wait();
  pdl_trigger();
#ifdef PIKO_EXP_NOTILE
  return;  // ablation: everything before the tile kernel
#endif
  const u64 frame = a.ctl->frame;
  const bool ovf = a.ctl->overflow_tag == frame + 1;
  if (a.status_out && blockIdx.x == 0 && tid < 32) {
    // the frame's control block (P, overflow tags, statistics) straight into
    // the host's pinned mirror: every field the host reads is final once the
    // AssignBin kernels are complete (this wait), so CTA 0 writes it here and
    // the PCIe writes drain under the tile work instead of trailing it (no
    // device-to-host copy on the stream, no last-CTA detection)
    constexpr int NW = (int)(offsetof(Control, digit_hist) / sizeof(u64));
    const volatile u64* src = reinterpret_cast<const volatile u64*>(a.ctl);
    u64* dst = reinterpret_cast<u64*>(a.status_out);
    for (int w = tid; w < NW; w += 32) dst[w] = src[w];
  }
  if (KEYS_ONLY && a.p2p_done) {  // P2P: rank 0 has finished reading this key slot
    if (tid == 0) p2p_wait_geq(a.p2p_done, (long long)a.epoch - 2, &a.ctl->p2p_timeout);
    __syncthreads();
  }
  TL_CTA(0);
  if (a.status_word && blockIdx.x == 0 && tid == 0)  // multi-GPU: overflow travels with the keys
    *a.status_word = ovf ? 0ull : a.status_ok;
  if (blockIdx.x == 0) {  // reset the next frame's double-buffered accumulators
    unsigned* h = &a.ctl->digit_hist[(frame + 1) & 1][0][0];
    for (int i = tid; i < MAX_PASSES * RX_RADIX; i += THREADS) h[i] = 0;
    if (tid == 0) a.ctl->n_live[(frame + 1) & 1] = 0;
    if (a.npass == 0 && tid == 0 && g.NB == 1) {  // single bin: CSR is [0, P]
      a.bin_start[0] = 0;
      a.bin_start[1] = ovf ? 0 : (int32_t)a.ctl->n_pairs;
    }
  }
  // next frame's look-back group arrival counters (every CTA a slice; only
  // the radix AssignBin uses them)
  for (int p = 0; p < (a.radix ? a.npass : 0); ++p) {
    uint32_t* ga = a.garrive + ((size_t)p * 2 + ((frame + 1) & 1)) * a.gcap;
    for (long long i = (long long)blockIdx.x * THREADS + tid; i < a.gcap; i += (long long)gridDim.x * THREADS)
      ga[i] = 0u;
  }
  // work-list sizes (single-bin grids have no bin scan: one job, bin 0)
  if (tid < NLIST) {
    unsigned n;
    if (a.npass > 0 && !ovf) n = a.ctl->list_n[tid];
    else if (ovf) n = (tid == LIST_EMPTY) ? (unsigned)a.owned : 0u;
    else {
      const bool one = a.owned > 0, any = a.ctl->n_pairs > 0;
      n = (tid == 1) ? (one && any) : (tid == LIST_EMPTY) ? (one && !any) : 0u;
    }
    s_ln[tid] = n;
  }
  __syncthreads();
  unsigned n_work = 0;
#pragma unroll
  for (int k = 0; k < LIST_EMPTY; ++k) n_work += s_ln[k];
  const unsigned n_frag = s_ln[0];
  const unsigned n_empty = a.skip_empty ? 0u : s_ln[LIST_EMPTY];  // (deferred resolve: background from the CSR)
  auto bin_range = [&](int b, int& rs, int& re) {
    if (a.npass == 0) { rs = 0; re = (int)a.ctl->n_pairs; return; }
    rs = a.bin_start[b];
    re = a.bin_start[b + 1];
  };
  // work item w -> bin, CSR sub-range, number of fragments of the bin (0:
  // unsplit), first fragment slot, fragment index.  Order (an LPT
  // approximation without a sort): whole bins of size class 1 (> 3/4 of a
  // fragment), then the fragments of split bins (balanced: a bin of n pairs
  // becomes nf = ceil(n / frag) fragments of n / nf pairs, no small
  // remainders), then size classes 2..4.  A bin's fragments are consecutive in
  // frag_list: fragment j of list position w keeps its key tile in slot w.
  auto work_item = [&](unsigned w, int& b, int& rs, int& re, int& nf, int& fs, int& fj) {
    fs = -1;
    fj = 0;
    const unsigned n1 = (a.npass == 0) ? 0u : s_ln[1];
    if (w >= n1 && w < n1 + n_frag) {
      const unsigned wf = w - n1;
      const int2 it = a.frag_list[wf];
      b = it.x;
      int s0, e0;
      bin_range(b, s0, e0);
      const long long n = e0 - s0;
      nf = (int)((n + a.frag - 1) / a.frag);
      rs = s0 + (int)((it.y * n) / nf);
      re = s0 + (int)(((it.y + 1) * n) / nf);
      fs = (int)wf - it.y;
      fj = it.y;
    } else if (w < n_work) {
      if (a.npass == 0) {
        b = 0;
      } else {  // size classes: list k >= 1 lives at bin_list[(k-1) NB]
        unsigned r;
        int k;
        if (w < n1) { r = w; k = 1; }
        else {
          r = w - n1 - n_frag;
          k = 2;
          while (r >= s_ln[k]) r -= s_ln[k++];
        }
        b = a.bin_list[(size_t)(k - 1) * g.NB + r];
      }
      bin_range(b, rs, re);
      nf = 0;
    } else {
      b = -1;
    }
  };
  auto empty_bin = [&](unsigned e) -> int {  // e < n_empty
    if (ovf) return g.rank + (int)e * g.nranks;
    if (a.npass == 0) return 0;
    return a.bin_list[(size_t)(LIST_EMPTY - 1) * g.NB + e];
  };

  // ---- LoadBalance schedule over the work list ----------------
  // thread 0 keeps the next item in registers one item ahead
  int q_bin = -1, q_s = 0, q_e = 0, q_nf = 0, q_fs = -1, q_fj = 0;
  unsigned q_tk = 0;
  bool have_q = false;  // thread 0: the q_* item is already looked up
  if (tid == 0) {
    // the first two items are static (blockIdx, blockIdx + grid): 2 x grid
    // same-address atomics at kernel start serialise at L2 for ~10 us; later
    // items come from the dynamic queue (its tickets start at 2 x grid)
    const unsigned t0 = blockIdx.x;
    q_tk = blockIdx.x + gridDim.x;
    int b0 = -1, s0 = 0, e0 = 0, nf0 = 0, fs0 = -1, fj0 = 0;
    work_item(t0, b0, s0, e0, nf0, fs0, fj0);
#if PIKO_EARLY_ITEM2
    // the second static item's lookups too, so its loads overlap the first's
    // (at the first item's start every CTA queries the lists at once)
    work_item(q_tk, q_bin, q_s, q_e, q_nf, q_fs, q_fj);
    have_q = true;
#endif
    s_bin = b0; s_rng[0] = s0; s_rng[1] = e0; s_rng[2] = nf0; s_rng[3] = fs0; s_rng[4] = fj0;
  }
  __syncthreads();
  // Pipeline prologue of an item: primIDs of the first TQ rounds and the
  // records of the first NSTAGE-1 rounds (cp.async).  For every item after the
  // first it is issued as soon as the previous item's raster has freed the
  // record stages, so it overlaps that item's queue pass and write-back.
  // entry i of the current item's list, -1 past its end
  auto prim_at = [&](int s_, int e_, int i) -> int { return s_ + i < e_ ? a.bin_prims[s_ + i] : -1; };
  int tq[TQ];
  auto prologue = [&](int s_, int e_) {
#pragma unroll
    for (int j = 0; j < TQ; ++j) tq[j] = prim_at(s_, e_, j * THREADS + tid);
#pragma unroll
    for (int j = 0; j < NSTAGE - 1; ++j) {
      if (tq[j] >= 0) {
        const int tj = tq[j];
        cp_async16(&sm.rec[j][tid][0], a.rec + rec_at(tj, 0, a.rec_stride));
        cp_async16(&sm.rec[j][tid][1], a.rec + rec_at(tj, 1, a.rec_stride));
        cp_async16(&sm.rec[j][tid][2], a.rec + rec_at(tj, 2, a.rec_stride));
      }
      cp_async_commit();
    }
  };
  bool pre = false;  // prologue of the current item already issued (CTA-uniform)
  for (;;) {
    const int b = s_bin;
    if (b < 0) break;
    const int s = s_rng[0], e = s_rng[1], nfrag = s_rng[2], fslot0 = s_rng[3], fidx = s_rng[4];
    TL_MARK(b, 0);
    if (tid == 0) {  // prefetch the next item
      if (!have_q) work_item(q_tk, q_bin, q_s, q_e, q_nf, q_fs, q_fj);
      have_q = false;
      if (q_bin >= 0) q_tk = 2u * gridDim.x + atomicAdd(&a.ctl->tile_next, 1u);
      s_nx[0] = q_bin; s_nx[1] = q_s; s_nx[2] = q_e;
    }
    const int bx = b % g.binsX, by = b / g.binsX;
    const int x0 = bx * BW, y0 = by * BH;
    const int x1 = min(x0 + BW, g.W) - 1, y1 = min(y0 + BH, g.H) - 1;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      const int p = tid + k * THREADS;
      if (p < NPX) {
        sm.key[p] = CLEAR_KEY;
        if (COV) s_cov[p] = 0;
      }
    }
    if (tid == 0) s_nbig = 0;
    __syncthreads();  // tile cleared before any warp rasterizes into it
    // Each warp streams its share of the bin's list (items s + k*THREADS +
    // warp*32 + lane) through its own cp.async pipeline: no CTA barrier until
    // the bin is done.  Tiny triangles: one thread loops over its pixels;
    // larger ones: warp-cooperative (triangle, pixel) expansion.
    TL_MARK(b, 5);  // tile cleared
    if (!pre) prologue(s, e);
    const int nround = (e - s + THREADS - 1) / THREADS;
    for (int k = 0; k < nround; ++k) {
      const int buf = k % NSTAGE;
      const int t_cur = tq[0];
      {  // issue round k + NSTAGE - 1, fetch the primIDs of round k + TQ
        const int tn = tq[NSTAGE - 1];
        if (tn >= 0) {
          const int nb = (k + NSTAGE - 1) % NSTAGE;
          cp_async16(&sm.rec[nb][tid][0], a.rec + rec_at(tn, 0, a.rec_stride));
          cp_async16(&sm.rec[nb][tid][1], a.rec + rec_at(tn, 1, a.rec_stride));
          cp_async16(&sm.rec[nb][tid][2], a.rec + rec_at(tn, 2, a.rec_stride));
        }
        cp_async_commit();
#pragma unroll
        for (int j = 0; j < TQ - 1; ++j) tq[j] = tq[j + 1];
        tq[TQ - 1] = prim_at(s, e, (k + TQ) * THREADS + tid);
      }
      cp_async_wait<NSTAGE - 1>();
      __syncwarp();  // warp-mates' records of round k are visible
      int rx0 = 0, ry0 = 0, w = 1, area = 0;
      if (t_cur >= 0) {
        const RecView r = unpack(sm.rec[buf][tid][0], sm.rec[buf][tid][1], sm.rec[buf][tid][2]);
        rx0 = max(r.px0, x0); ry0 = max(r.py0, y0);
        w = min(r.px1, x1) - rx0 + 1;
        const int h = min(r.py1, y1) - ry0 + 1;
        area = w * h;
#ifdef PIKO_EXP_NORASTER
        area = 0;
#endif
        if (area <= TINY_AREA) {
#ifdef PIKO_EXP_NORASTER
          if (r.X0 == 123456789) sm.key[0] = t_cur;
#else
#if PIKO_TINY32
          if (r.small) {
            // small triangle (bbox extent < 2^15 subpixels): the three edge
            // functions at the clipped rect's first sample, then stepped by
            // -256 A per pixel and +256 B per row -- the same exact integer
            // values as eval_pre (every sample lies in the bbox, so each true
            // value fits int32 and the wrapped unsigned sums are exact) without
            // its 64-bit constants; depth from the same fma chain
            const int dx0 = 256 * rx0 + 128 - r.X0, dy0 = 256 * ry0 + 128 - r.Y0;
            const unsigned A0 = (unsigned)(r.Y1 - r.Y0), B0 = (unsigned)(r.X1 - r.X0);
            const unsigned A1 = (unsigned)(r.Y2 - r.Y1), B1 = (unsigned)(r.X2 - r.X1);
            const unsigned A2 = (unsigned)(r.Y0 - r.Y2), B2 = (unsigned)(r.X0 - r.X2);
            unsigned q0 = B0 * (unsigned)dy0 - A0 * (unsigned)dx0;
            unsigned q1 = B1 * (unsigned)(dy0 + r.Y0 - r.Y1) - A1 * (unsigned)(dx0 + r.X0 - r.X1);
            unsigned q2 = B2 * (unsigned)(dy0 + r.Y0 - r.Y2) - A2 * (unsigned)(dx0 + r.X0 - r.X2);
            const int th0 = tl_thr(r.X0, r.Y0, r.X1, r.Y1), th1 = tl_thr(r.X1, r.Y1, r.X2, r.Y2);
            const int th2 = tl_thr(r.X2, r.Y2, r.X0, r.Y0);
            int p0 = (ry0 - y0) * BW + (rx0 - x0);
            for (int yy = 0; yy < h; ++yy) {
              unsigned e0 = q0, e1 = q1, e2 = q2;
              for (int xx = 0; xx < w; ++xx) {
                if ((int)e0 > th0 && (int)e1 > th1 && (int)e2 > th2) {
                  if (COV) atomicAdd(&s_cov[p0 + xx], 1u);
                  const float z = __fmaf_rn(r.za, __int2float_rn(dx0 + 256 * xx),
                                            __fmaf_rn(r.zb, __int2float_rn(dy0 + 256 * yy), r.zw0));
                  if (z >= 0.0f && z <= 1.0f) {
                    const u64 key = ((u64)(__float_as_uint(z) & 0x7FFFFFFFu) << 32) | (unsigned)t_cur;
                    atomicMin(&sm.key[p0 + xx], key);
                    if (fwd) facc = __fadd_rn(facc, shader_work(fwd, key_depth(key)));
                  }
                }
                e0 -= 256u * A0; e1 -= 256u * A1; e2 -= 256u * A2;
              }
              q0 += 256u * B0; q1 += 256u * B1; q2 += 256u * B2;
              p0 += BW;
            }
          } else
#endif
          {
          const TriEval ev = prepare(r);
          for (int y = ry0; y < ry0 + h; ++y)
            for (int x = rx0; x < rx0 + w; ++x) {
              bool cov;
              const u64 key = eval_pre(ev, 256 * x + 128, 256 * y + 128, t_cur, cov);
              const int p = (y - y0) * BW + (x - x0);
              if (COV && cov) atomicAdd(&s_cov[p], 1u);
#ifndef PIKO_EXP_NOATOM
              if (key != CLEAR_KEY) {
                atomicMin(&sm.key[p], key);
                if (fwd) facc = __fadd_rn(facc, shader_work(fwd, key_depth(key)));
              }
#else
              if (key == 12345) sm.key[p] = key;
#endif
            }
          }
#endif
          area = 0;
        } else {
          const int slot = atomicAdd(&s_nbig, 1);
          if (slot < TileSmem<BW, BH, THREADS>::BIGQ) {
            const TriEval ev = prepare(r);
            auto& Q = sm.q;
            Q.X0[slot] = ev.X0; Q.Y0[slot] = ev.Y0;
            Q.A0[slot] = ev.A0; Q.B0[slot] = ev.B0; Q.A1[slot] = ev.A1; Q.B1[slot] = ev.B1;
            Q.A2[slot] = ev.A2; Q.B2[slot] = ev.B2; Q.K1[slot] = ev.K1; Q.K2[slot] = ev.K2;
            Q.thr[slot] = (ev.thr0 ? 1 : 0) | (ev.thr1 ? 2 : 0) | (ev.thr2 ? 4 : 0) | (ev.small ? 8 : 0);
            Q.zw0[slot] = ev.zw0; Q.za[slot] = ev.za; Q.zb[slot] = ev.zb;
            Q.invw[slot] = __frcp_rn((float)((w + QSEG - 1) / QSEG));  // 1 / segments per row
            Q.t[slot] = t_cur; Q.rx0[slot] = rx0; Q.ry0[slot] = ry0; Q.w[slot] = w;
            Q.pre[slot] = (unsigned)(h * ((w + QSEG - 1) / QSEG));  // segments; prefix at the end of the bin
            area = 0;
          } else if (a.ovq && slot - TileSmem<BW, BH, THREADS>::BIGQ < OVQ_CAP) {
            // queue full: spill the prepared entry to this CTA's global overflow
            // region (L2); drained by all threads after the main loop, so no
            // warp is left rasterizing alone while the others wait
            const TriEval ev = prepare(r);
            int4* q = a.ovq + ((size_t)blockIdx.x * OVQ_CAP + (slot - TileSmem<BW, BH, THREADS>::BIGQ)) * 6;
            const int thr = (ev.thr0 ? 1 : 0) | (ev.thr1 ? 2 : 0) | (ev.thr2 ? 4 : 0) | (ev.small ? 8 : 0);
            q[0] = make_int4(ev.X0, ev.Y0, ev.A0, ev.B0);
            q[1] = make_int4(ev.A1, ev.B1, ev.A2, ev.B2);
            q[2] = make_int4((int)(unsigned)ev.K1, (int)(ev.K1 >> 32), (int)(unsigned)ev.K2, (int)(ev.K2 >> 32));
            q[3] = make_int4(thr, __float_as_int(ev.zw0), __float_as_int(ev.za), __float_as_int(ev.zb));
            q[4] = make_int4(__float_as_int(__frcp_rn((float)((w + QSEG - 1) / QSEG))), t_cur, rx0, ry0);
            q[5] = make_int4(w, h * ((w + QSEG - 1) / QSEG), 0, 0);
            area = 0;
          }  // both full: this one takes the warp-cooperative path
        }
      }
      if (__any_sync(0xffffffffu, area > 0)) {  // queue overflow: warp-cooperative
        unsigned incl = (unsigned)area;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += v;
        }
        const unsigned total = __shfl_sync(0xffffffffu, incl, 31);
        for (unsigned base = 0; base < total; base += 32) {
          const unsigned item = base + lane;
          int src = 0;  // first lane whose inclusive prefix exceeds item
#pragma unroll
          for (int st = 16; st >= 1; st >>= 1) {
            const unsigned v = __shfl_sync(0xffffffffu, incl, src + st - 1);
            if (v <= item) src += st;
          }
          src = min(src, 31);
          const unsigned incl_s = __shfl_sync(0xffffffffu, incl, src);
          const int area_s = __shfl_sync(0xffffffffu, area, src);
          const int rx0_s = __shfl_sync(0xffffffffu, rx0, src);
          const int ry0_s = __shfl_sync(0xffffffffu, ry0, src);
          const int w_s = __shfl_sync(0xffffffffu, w, src);
          const int t_s = __shfl_sync(0xffffffffu, t_cur, src);
          if (item < total) {
            const int off = (int)(item - (incl_s - (unsigned)area_s));
            const int y = ry0_s + off / w_s, x = rx0_s + off % w_s;
            const int sl = warp * 32 + src;
            const RecView rs = unpack(sm.rec[buf][sl][0], sm.rec[buf][sl][1], sm.rec[buf][sl][2]);
            bool cov;
            const u64 key = eval_key(rs, 256 * x + 128, 256 * y + 128, t_s, cov);
            const int p = (y - y0) * BW + (x - x0);
            if (COV && cov) atomicAdd(&s_cov[p], 1u);
            if (key != CLEAR_KEY) {
              atomicMin(&sm.key[p], key);
              if (fwd) facc = __fadd_rn(facc, shader_work(fwd, key_depth(key)));
            }
          }
        }
      }
      __syncwarp();  // round k's slots are free for round k + NSTAGE
    }
    TL_MARK(b, 6);  // rounds issued/rasterized
    cp_async_wait<0>();
    __syncthreads();
    TL_MARK(b, 7);  // all records consumed
    // record stages are free: start the next item's loads now
    pre = s_nx[0] >= 0;
    if (pre) prologue(s_nx[1], s_nx[2]);
    // queued triangles: all threads over the flattened (triangle, pixel) items
    auto drain = [&](const int nq) {
      {
        auto& Q = sm.q;
        // exclusive prefix of the clipped areas (one entry per thread)
        const unsigned ar = tid < nq ? Q.pre[tid] : 0u;
        unsigned inc = ar;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned v = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += v;
        }
        __shared__ unsigned s_qw[THREADS / 32];
        if (lane == 31) s_qw[warp] = inc;
        __syncthreads();
        unsigned wbase = 0, tot = 0;
#pragma unroll
        for (int w2 = 0; w2 < THREADS / 32; ++w2) {
          const unsigned v = s_qw[w2];
          wbase += (w2 < warp) ? v : 0u;
          tot += v;
        }
        if (tid < nq) Q.pre[tid] = wbase + inc - ar;
        if (tid == 0) Q.pre[nq] = tot;
        __syncthreads();
        // warp-contiguous items.  qw = the entry holding the warp's first item
        // (monotone): lanes load the next 32 entry starts and a ballot advances
        // qw (pre is strictly increasing, so the mask is a prefix).  Every
        // entry covers >= 1 item (a row segment of <= QSEG pixels), so the warp's 32 items lie in
        // entries qw .. qw+31 and each lane finds its own with a 5-step shuffle
        // search over the loaded starts -- no serial per-warp search.
        int qw = 0;
        for (unsigned base = (unsigned)warp * 32; base < tot; base += THREADS) {
          unsigned pk;
          for (;;) {
            const int k = qw + 1 + lane;
            pk = k <= nq ? Q.pre[k] : 0xFFFFFFFFu;
            const unsigned m = __ballot_sync(0xffffffffu, pk <= base);
            qw += __popc(m);
            if (m != 0xFFFFFFFFu) {
              if (m) pk = (qw + 1 + lane <= nq) ? Q.pre[qw + 1 + lane] : 0xFFFFFFFFu;
              break;
            }
          }
          const unsigned i = base + lane;
          int c = 0;  // entries after qw starting at or before item i
#pragma unroll
          for (int st = 16; st >= 1; st >>= 1) {
            const unsigned v = __shfl_sync(0xffffffffu, pk, c + st - 1);
            if (v <= i) c += st;
          }
          if (i >= tot) continue;
          const int q = qw + c;
          const unsigned off = i - Q.pre[q];
          const int wq = Q.w[q], spr = (wq + QSEG - 1) / QSEG;
          const int row = __float2int_rz(((float)off + 0.5f) * Q.invw[q]);  // exact: off < 2^12
          const int seg = (int)off - row * spr;
          const int xs = Q.rx0[q] + seg * QSEG, y = Q.ry0[q] + row;
          const int nseg = min(QSEG, wq - seg * QSEG);  // pixels of this segment
          TriEval ev;
          ev.X0 = Q.X0[q]; ev.Y0 = Q.Y0[q];
          ev.A0 = Q.A0[q]; ev.B0 = Q.B0[q]; ev.A1 = Q.A1[q]; ev.B1 = Q.B1[q];
          ev.A2 = Q.A2[q]; ev.B2 = Q.B2[q]; ev.K1 = Q.K1[q]; ev.K2 = Q.K2[q];
          const int th = Q.thr[q];
          ev.thr0 = (th & 1) ? -1 : 0; ev.thr1 = (th & 2) ? -1 : 0; ev.thr2 = (th & 4) ? -1 : 0;
          ev.small = (th >> 3) & 1;
          ev.zw0 = Q.zw0[q]; ev.za = Q.za[q]; ev.zb = Q.zb[q];
          const int tq = Q.t[q];
#pragma unroll
          for (int u = 0; u < QSEG; ++u) {
            if (u >= nseg) break;
            const int x = xs + u;
            bool cov;
            const u64 key = eval_pre(ev, 256 * x + 128, 256 * y + 128, tq, cov);
            const int p = (y - y0) * BW + (x - x0);
            if (COV && cov) atomicAdd(&s_cov[p], 1u);
            if (key != CLEAR_KEY) {
              atomicMin(&sm.key[p], key);
              if (fwd) facc = __fadd_rn(facc, shader_work(fwd, key_depth(key)));
            }
          }
        }
        __syncthreads();
      }
    };
    {
      constexpr int BIGQ = TileSmem<BW, BH, THREADS>::BIGQ;
      const int nbig = s_nbig;
      if (nbig > 0) drain(min(nbig, BIGQ));
      // spilled entries, BIGQ at a time through the same shared-memory queue
      const int nov = a.ovq ? min(max(nbig - BIGQ, 0), OVQ_CAP) : 0;
      for (int o0 = 0; o0 < nov; o0 += BIGQ) {
        const int nq = min(BIGQ, nov - o0);
        if (tid < nq) {
          const int4* q = a.ovq + ((size_t)blockIdx.x * OVQ_CAP + o0 + tid) * 6;
          const int4 q0 = q[0], q1 = q[1], q2 = q[2], q3 = q[3], q4 = q[4], q5 = q[5];
          auto& Q = sm.q;
          Q.X0[tid] = q0.x; Q.Y0[tid] = q0.y; Q.A0[tid] = q0.z; Q.B0[tid] = q0.w;
          Q.A1[tid] = q1.x; Q.B1[tid] = q1.y; Q.A2[tid] = q1.z; Q.B2[tid] = q1.w;
          Q.K1[tid] = (long long)(((unsigned long long)(unsigned)q2.y << 32) | (unsigned)q2.x);
          Q.K2[tid] = (long long)(((unsigned long long)(unsigned)q2.w << 32) | (unsigned)q2.z);
          Q.thr[tid] = q3.x; Q.zw0[tid] = __int_as_float(q3.y); Q.za[tid] = __int_as_float(q3.z);
          Q.zb[tid] = __int_as_float(q3.w);
          Q.invw[tid] = __int_as_float(q4.x); Q.t[tid] = q4.y; Q.rx0[tid] = q4.z; Q.ry0[tid] = q4.w;
          Q.w[tid] = q5.x; Q.pre[tid] = (unsigned)q5.y;
        }
        __syncthreads();  // batch staged (the previous drain ended with a barrier)
        drain(nq);
      }
    }
    TL_MARK(b, 1);

    // ---- write-back ----------------------------------------------------------
    const int job = (b - g.rank) / g.nranks;
    if (nfrag == 0) {
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
        const int p = tid + k * THREADS;
        if (p >= NPX) continue;
        const int x = x0 + (p % BW), y = y0 + (p / BW);
        if (!KEYS_ONLY && (x > x1 || y > y1)) continue;
        store_pixel<COV, KEYS_ONLY>(a, L, job, p, NPX, x, y, sm.key[p], COV ? s_cov[p] : 0u);
      }
    } else {
      // fragment of a split bin: its key tile goes to its own slot with plain
      // coalesced stores (no atomics); the last fragment to arrive takes the
      // per-pixel minimum over the bin's slots and writes the bin
      const int myslot = fslot0 + fidx;
#pragma unroll
      for (int k = 0; k < PPT; ++k) {
        const int p = tid + k * THREADS;
        if (p >= NPX) continue;
        a.fkey[(size_t)myslot * NPX + p] = sm.key[p];
        if (COV && s_cov[p]) atomicAdd(&a.gcov[(size_t)b * NPX + p], s_cov[p]);
      }
      __threadfence();
      __syncthreads();
      if (tid == 0) {
        const unsigned done = atomicAdd(&a.arrive[b], 1u) + 1u;
        s_last = done == (unsigned)nfrag;
        if (s_last) a.arrive[b] = 0u;  // ready for the next frame
      }
      __syncthreads();
      if (s_last) {
        __threadfence();
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          const int p = tid + k * THREADS;
          if (p >= NPX) continue;
          const int x = x0 + (p % BW), y = y0 + (p / BW);
          if (!KEYS_ONLY && (x > x1 || y > y1)) continue;
          u64 key = sm.key[p];
          for (int f0 = 0; f0 < nfrag; f0 += 4) {  // 4 slot loads in flight
            u64 kv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
              kv[u] = (f0 + u < nfrag && fslot0 + f0 + u != myslot)
                          ? __ldcg(&a.fkey[(size_t)(fslot0 + f0 + u) * NPX + p]) : CLEAR_KEY;
#pragma unroll
            for (int u = 0; u < 4; ++u) key = kv[u] < key ? kv[u] : key;
          }
          const unsigned cv = COV ? __ldcg(&a.gcov[(size_t)b * NPX + p]) : 0u;
          if (COV) a.gcov[(size_t)b * NPX + p] = 0u;
          store_pixel<COV, KEYS_ONLY>(a, L, job, p, NPX, x, y, key, cv);
        }
      }
    }
    TL_MARK(b, 2);
    if (tid == 0 && b < 8192) { g_tl_extra(b, e - s, blockIdx.x); }
    __syncthreads();  // keys consumed before the next bin reinitialises them
    if (tid == 0) { s_bin = q_bin; s_rng[0] = q_s; s_rng[1] = q_e; s_rng[2] = q_nf; s_rng[3] = q_fs; s_rng[4] = q_fj; }
    __syncthreads();
  }

  TL_CTA(1);
  // ---- empty bins: background only, no shared memory, no barriers ------------
  // every warp pulls groups of EMPTY_GROUP bins from a second queue
  // (one queue ticket per CTA for THREADS/32 groups: per-warp tickets on one
  // address serialised at L2)
#ifdef PIKO_EXP_NOEMPTY
  if (false)
#endif
  if (a.early_empty && !ovf) empty_pass();  // what the early CTAs left of the same queue
  else
  for (;;) {
    __syncthreads();
    if (tid == 0) s_etk = atomicAdd(&a.ctl->empty_next, 1u);
    __syncthreads();
    const unsigned e0 = (s_etk * (THREADS / 32) + warp) * EMPTY_GROUP;
    if (s_etk * (THREADS / 32) * EMPTY_GROUP >= n_empty) break;
    // the group's bin ids in one round trip (lane l loads entry e0 + l), not
    // one dependent load per bin
    const int bl = (lane < EMPTY_GROUP && e0 + lane < n_empty) ? empty_bin(e0 + lane) : 0;
    for (unsigned e = e0; e < min(e0 + EMPTY_GROUP, n_empty); ++e) {
      const int b = __shfl_sync(0xffffffffu, bl, (int)(e - e0));
      const int x0 = (b % g.binsX) * BW, y0 = (b / g.binsX) * BH;
      const int x1 = min(x0 + BW, g.W) - 1, y1 = min(y0 + BH, g.H) - 1;
      const int job = (b - g.rank) / g.nranks;
      for (int p = lane; p < NPX; p += 32) {
        const int x = x0 + (p % BW), y = y0 + (p / BW);
        if (!KEYS_ONLY && (x > x1 || y > y1)) continue;
        store_pixel<COV, KEYS_ONLY>(a, L, job, p, NPX, x, y, CLEAR_KEY, 0u);
      }
    }
  }
  TL_CTA(2);
  if (fwd) shader_sink(a.sc, facc);
  if (KEYS_ONLY && a.p2p_flag) {
    // P2P: every CTA's key stores (straight into rank 0's memory over NVLink)
    // are made visible system-wide before it is counted; the last CTA counted
    // raises this rank's arrival flag at rank 0 (release, system scope)
    __syncthreads();
    if (tid == 0) {
      __threadfence_system();
      const u64 t = atomicAdd(&a.ctl->p2p_arrive, 1ull);
      if ((t + 1) % gridDim.x == 0) {
        __threadfence_system();
        st_release_sys64(a.p2p_flag, a.epoch);
      }
    }
  }
}

#ifndef PIKO_TILE_TU
// ---------------------------------------------------------------------------
// FreePipe (NEXT-3 design alternative): the whole pipeline fused
// into one kernel with static (DirectMap) triangle -> thread mapping; fragments
// meet in a full-screen key buffer through 64-bit atomicMin (deterministic:
// the min is order independent), then one resolve pass shades.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_freepipe(FreePipeArgs a) {
  pdl_wait();
  pdl_trigger();
  const int fwd = a.sc.forward ? a.sc.iters : 0;  // forward shader cost per fragment
  float facc = 0.0f;
  constexpr int TPT = 4;
  const long long tb = (long long)blockIdx.x * (256 * TPT) + threadIdx.x;
  int vi[TPT][3];
#pragma unroll
  for (int k = 0; k < TPT; ++k) {
    const long long t = tb + k * 256;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      vi[k][c] = t < a.n_tris ? __ldg(a.idx + 3 * t + c) : -1;
      if (a.xv && vi[k][c] >= a.xv_cap) vi[k][c] = -1;
    }
  }
  int4 cv[TPT][3];
#pragma unroll
  for (int k = 0; k < TPT; ++k)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      cv[k][c] = vi[k][c] < 0 ? make_int4(VX_CULLED, 0, 0, 0)
                 : a.xv     ? __ldg(a.xv + vi[k][c])
                            : transform_vertex(load_pos(a.verts, vi[k][c]), a.M, a.W, a.H);
#pragma unroll 1
  for (int k = 0; k < TPT; ++k) {
    const long long t = tb + k * 256;
    Tri o;
    if (t >= a.n_tris ||
        !setup_tri(cv[k][0], cv[k][1], cv[k][2], vi[k][0], vi[k][1], vi[k][2], a.W, a.H, o))
      continue;
    const float dx1 = __int2float_rn(o.X1 - o.X0), dy1 = __int2float_rn(o.Y1 - o.Y0);
    const float dx2 = __int2float_rn(o.X2 - o.X0), dy2 = __int2float_rn(o.Y2 - o.Y0);
    const float dz1 = __fsub_rn(o.zw1, o.zw0), dz2 = __fsub_rn(o.zw2, o.zw0);
    const float inv = __frcp_rn(__ll2float_rn(o.area2));
    RecView r;
    r.X0 = o.X0; r.Y0 = o.Y0; r.X1 = o.X1; r.Y1 = o.Y1; r.X2 = o.X2; r.Y2 = o.Y2;
    r.zw0 = o.zw0;
    r.za = __fmul_rn(__fmaf_rn(dz1, dy2, -__fmul_rn(dz2, dy1)), inv);
    r.zb = __fmul_rn(__fmaf_rn(dz2, dx1, -__fmul_rn(dz1, dx2)), inv);
    r.px0 = o.px0; r.py0 = o.py0; r.px1 = o.px1; r.py1 = o.py1;
    r.small = o.small;
    const TriEval ev = prepare(r);
    for (int y = o.py0; y <= o.py1; ++y)
      for (int x = o.px0; x <= o.px1; ++x) {
        bool cov;
        const u64 key = eval_pre(ev, 256 * x + 128, 256 * y + 128, (int)t, cov);
        const size_t p = (size_t)y * a.W + x;
        if (a.cov && cov) atomicAdd(&a.cov[p], 1u);
        if (key != CLEAR_KEY) {
          atomicMin(&a.keys[p], key);
          if (fwd) facc = __fadd_rn(facc, shader_work(fwd, key_depth(key)));
        }
      }
  }
  if (fwd) shader_sink(a.sc, facc);
}

__global__ void __launch_bounds__(256) k_fp_resolve(const __grid_constant__ FreePipeArgs a) {
  pdl_wait();
  pdl_trigger();
  const long long p = (long long)blockIdx.x * 256 + threadIdx.x;
  if (p >= (long long)a.W * a.H) return;
  const int x = (int)(p % a.W), y = (int)(p / a.W);
  const u64 key = a.keys[p];
  a.keys[p] = CLEAR_KEY;  // ready for the next frame
  float L[3];
  normalise_light(a.light, L);
  float4 c = make_float4(0.f, 0.f, 0.f, 0.f);
  float depth = 1.0f;
  int prim = -1;
  if (key != CLEAR_KEY) {
    prim = (int)(unsigned)(key & 0xFFFFFFFFu);
    depth = __uint_as_float((unsigned)(key >> 32));
    c = shade(a.verts, a.xv, &a.M, a.idx, a.W, a.H, L, prim, 256 * x + 128, 256 * y + 128);
    if (a.sc.iters && !a.sc.forward) shader_sink(a.sc, shader_work(a.sc.iters, depth));
  }
  reinterpret_cast<float4*>(a.out_rgba)[p] = c;
  a.out_depth[p] = depth;
  a.out_primid[p] = prim;
}

// ---------------------------------------------------------------------------
// Baseline (NEXT-3 design alternative): the five
// stages as separate kernels with full-screen bins, each reading its input
// from and writing its output to off-chip memory.  Rasterizer: thread per
// triangle, fragments appended to a global buffer (count, warp-aggregated
// reservation, emit); Fragment Shader: thread per fragment; Depth Test:
// 64-bit atomicMin per fragment; Composite: the winning fragment of each
// pixel writes it, then a per-pixel pass writes background and clears the
// depth buffer.  Same arithmetic as the binned path: bit-identical frames.
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool bl_setup(const BaselineArgs& a, long long t, TriEval& ev, int& px0,
                                         int& py0, int& px1, int& py1) {
  if (t >= a.n_tris) return false;
  int vi[3];
  int4 cv[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    vi[c] = __ldg(a.idx + 3 * t + c);
    cv[c] = vi[c] < a.xv_cap ? __ldg(a.xv + vi[c]) : make_int4(VX_CULLED, 0, 0, 0);
  }
  Tri o;
  if (!setup_tri(cv[0], cv[1], cv[2], vi[0], vi[1], vi[2], a.W, a.H, o)) return false;
  const float dx1 = __int2float_rn(o.X1 - o.X0), dy1 = __int2float_rn(o.Y1 - o.Y0);
  const float dx2 = __int2float_rn(o.X2 - o.X0), dy2 = __int2float_rn(o.Y2 - o.Y0);
  const float dz1 = __fsub_rn(o.zw1, o.zw0), dz2 = __fsub_rn(o.zw2, o.zw0);
  const float inv = __frcp_rn(__ll2float_rn(o.area2));
  RecView r;
  r.X0 = o.X0; r.Y0 = o.Y0; r.X1 = o.X1; r.Y1 = o.Y1; r.X2 = o.X2; r.Y2 = o.Y2;
  r.zw0 = o.zw0;
  r.za = __fmul_rn(__fmaf_rn(dz1, dy2, -__fmul_rn(dz2, dy1)), inv);
  r.zb = __fmul_rn(__fmaf_rn(dz2, dx1, -__fmul_rn(dz1, dx2)), inv);
  r.px0 = o.px0; r.py0 = o.py0; r.px1 = o.px1; r.py1 = o.py1;
  r.small = o.small;
  ev = prepare(r);
  px0 = o.px0; py0 = o.py0; px1 = o.px1; py1 = o.py1;
  return true;
}

__global__ void __launch_bounds__(256) k_bl_raster(BaselineArgs a) {
  pdl_wait();
  pdl_trigger();
  const long long t = (long long)blockIdx.x * 256 + threadIdx.x;
  const int lane = threadIdx.x & 31;
  TriEval ev;
  int px0 = 0, py0 = 0, px1 = -1, py1 = -1;
  const bool live = bl_setup(a, t, ev, px0, py0, px1, py1);
  // pass 1: count this triangle's fragments (covered, depth in range)
  unsigned n = 0;
  if (live)
    for (int y = py0; y <= py1; ++y)
      for (int x = px0; x <= px1; ++x) {
        bool cov;
        const u64 key = eval_pre(ev, 256 * x + 128, 256 * y + 128, (int)t, cov);
        if (a.cov && cov) atomicAdd(&a.cov[(size_t)y * a.W + x], 1u);
        n += key != CLEAR_KEY;
      }
  // one reservation per warp
  unsigned incl = n;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const unsigned tot = __shfl_sync(0xffffffffu, incl, 31);
  u64 base = 0;
  if (lane == 31 && tot) base = atomicAdd(a.n_frag, (u64)tot);
  base = __shfl_sync(0xffffffffu, base, 31) + (incl - n);
  // pass 2: emit (fragments beyond the capacity are counted, not stored)
  if (n)
    for (int y = py0; y <= py1; ++y)
      for (int x = px0; x <= px1; ++x) {
        bool cov;
        const u64 key = eval_pre(ev, 256 * x + 128, 256 * y + 128, (int)t, cov);
        if (key == CLEAR_KEY) continue;
        if ((long long)base < a.frag_cap) {
          a.frag_key[base] = key;
          a.frag_px[base] = (uint32_t)((size_t)y * a.W + x);
        }
        ++base;
      }
}

__global__ void __launch_bounds__(256) k_bl_fs(BaselineArgs a) {
  pdl_wait();
  pdl_trigger();
  float L[3];
  normalise_light(a.light, L);
  const long long n = min((long long)*a.n_frag, a.frag_cap);
  const int fwd = a.sc.forward ? a.sc.iters : 0;
  float facc = 0.0f;
  for (long long i = (long long)blockIdx.x * 256 + threadIdx.x; i < n; i += (long long)gridDim.x * 256) {
    const u64 key = a.frag_key[i];
    const uint32_t p = a.frag_px[i];
    const int x = (int)(p % (uint32_t)a.W), y = (int)(p / (uint32_t)a.W);
    a.frag_rgba[i] = shade(a.verts, a.xv, &a.M, a.idx, a.W, a.H, L, (int)(unsigned)(key & 0xFFFFFFFFu),
                           256 * x + 128, 256 * y + 128);
    if (fwd) facc = __fadd_rn(facc, shader_work(fwd, key_depth(key)));
  }
  if (fwd) shader_sink(a.sc, facc);
}

__global__ void __launch_bounds__(256) k_bl_depth(BaselineArgs a) {
  pdl_wait();
  pdl_trigger();
  const long long n = min((long long)*a.n_frag, a.frag_cap);
  for (long long i = (long long)blockIdx.x * 256 + threadIdx.x; i < n; i += (long long)gridDim.x * 256)
    atomicMin(&a.keys[a.frag_px[i]], a.frag_key[i]);
}

__global__ void __launch_bounds__(256) k_bl_composite(BaselineArgs a) {
  pdl_wait();
  pdl_trigger();
  const long long n = min((long long)*a.n_frag, a.frag_cap);
  for (long long i = (long long)blockIdx.x * 256 + threadIdx.x; i < n; i += (long long)gridDim.x * 256) {
    const u64 key = a.frag_key[i];
    const uint32_t p = a.frag_px[i];
    if (a.keys[p] != key) continue;  // keys are unique per pixel: one winner
    reinterpret_cast<float4*>(a.out_rgba)[p] = a.frag_rgba[i];
    a.out_depth[p] = key_depth(key);
    a.out_primid[p] = (int)(unsigned)(key & 0xFFFFFFFFu);
    if (a.sc.iters && !a.sc.forward) shader_sink(a.sc, shader_work(a.sc.iters, key_depth(key)));
  }
}

__global__ void __launch_bounds__(256) k_bl_clear(BaselineArgs a) {
  pdl_wait();
  pdl_trigger();
  const long long p = (long long)blockIdx.x * 256 + threadIdx.x;
  if (p >= (long long)a.W * a.H) return;
  if (a.keys[p] == CLEAR_KEY) {
    reinterpret_cast<float4*>(a.out_rgba)[p] = make_float4(0.f, 0.f, 0.f, 0.f);
    a.out_depth[p] = 1.0f;
    a.out_primid[p] = -1;
  }
  a.keys[p] = CLEAR_KEY;  // ready for the next frame
}

// ---------------------------------------------------------------------------
// K7 (multi-GPU rank 0): resolve gathered tile keys -> shaded frame
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_resolve(const __grid_constant__ ResolveArgs a) {
  pdl_wait();
  pdl_trigger();
  const Grid g = a.g;
  const int x = blockIdx.x * 32 + (threadIdx.x & 31);
  const int y = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (a.p2p_flags) {  // P2P: every rank's keys have arrived (acquire, system scope)
    if (threadIdx.x == 0)
      for (int q = 0; q < g.nranks; ++q) p2p_wait_geq(a.p2p_flags + q, (long long)a.epoch, a.p2p_timeout);
    __syncthreads();
  }
  const bool in = x < g.W && y < g.H;
  u64 key = CLEAR_KEY;
  int bw = 0, bh = 0;
  if (in) {
    bw = 1 << g.bw_log2; bh = 1 << g.bh_log2;
    const int b = (y >> g.bh_log2) * g.binsX + (x >> g.bw_log2);
    const int r = b % g.nranks, k = b / g.nranks;
    const int p = (y & (bh - 1)) * bw + (x & (bw - 1));
    const size_t rs = a.rank_stride ? (size_t)a.rank_stride : (size_t)a.owned_max * (size_t)(bw * bh);
    // written by peers: bypass L1
    key = __ldcg(&a.all_keys[(size_t)r * rs + (size_t)k * (size_t)(bw * bh) + p]);
  }
  if (a.status && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
    // a rank that overflowed its pair capacity sent empty bins: rank 0's
    // frame is incomplete and its host reports PIKO_ECAPACITY
    bool bad = false;
    for (int q = 0; q < a.nstatus; ++q) bad |= __ldcg(a.status + (size_t)q * a.status_stride) != a.status_ok;
    if (bad) a.ctl->peer_overflow = a.ctl->frame + 1;
  }
  if (a.p2p_flags) {  // this CTA's keys are read: the last CTA releases the slot
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned nblk = gridDim.x * gridDim.y;
      __threadfence();  // this CTA's key loads are ordered before its ticket (WAR vs the peers)
      const unsigned long long t = atomicAdd(a.p2p_count, 1ull);
      if ((t + 1) % nblk == 0) st_release_sys64(a.p2p_done, a.epoch);
    }
  }
  if (!in) return;
  float L[3];
  normalise_light(a.light, L);
  const size_t o = (size_t)y * g.W + x;
  float4 c = make_float4(0.f, 0.f, 0.f, 0.f);
  float depth = 1.0f;
  int prim = -1;
  if (key != CLEAR_KEY) {
    prim = (int)(unsigned)(key & 0xFFFFFFFFu);
    depth = __uint_as_float((unsigned)(key >> 32));
    c = shade(a.verts, a.xv, &a.M, a.idx, g.W, g.H, L, prim, 256 * x + 128, 256 * y + 128);
    if (a.sc.iters && !a.sc.forward) shader_sink(a.sc, shader_work(a.sc.iters, depth));
  }
  reinterpret_cast<float4*>(a.out_rgba)[o] = c;
  a.out_depth[o] = depth;
  a.out_primid[o] = prim;
}

// ---------------------------------------------------------------------------
// k_shade: single-GPU deferred resolve (Composite + Fragment Shader of the
// winners).  k_tile left the packed (depth, primID) key of every
// pixel in bin-major tiles; each thread shades a quad of 4 pixels of a row
// with the loads of all 4 in flight together, then writes RGBA, depth and
// primID with vector stores.  Full occupancy (no shared memory): the
// dependent gathers of shading are hidden across warps instead of sitting on
// k_tile's per-bin critical path.
// ---------------------------------------------------------------------------
#ifndef PIKO_SHADE_QUAD
#define PIKO_SHADE_QUAD 4
#endif
constexpr int SHADE_QUAD = PIKO_SHADE_QUAD;  // pixels of a row per k_shade thread (1 or 4)
__global__ void __launch_bounds__(256) k_shade(const __grid_constant__ ResolveArgs a) {
  pdl_wait();
  pdl_trigger();
  const Grid g = a.g;
  const int qx = (g.W + SHADE_QUAD - 1) / SHADE_QUAD;
  const long long q = (long long)blockIdx.x * 256 + threadIdx.x;
  if (q >= (long long)qx * g.H) return;
  const int y = (int)(q / qx), x0 = (int)(q % qx) * SHADE_QUAD;
  const int bw = 1 << g.bw_log2, bh = 1 << g.bh_log2;
  const int b = (y >> g.bh_log2) * g.binsX + (x0 >> g.bw_log2);
  const int p = (y & (bh - 1)) * bw + (x0 & (bw - 1));
  // bins are >= 8 px wide and x0 % 4 == 0: the quad is 4 consecutive keys of one bin row
  u64 key[SHADE_QUAD];
  if constexpr (SHADE_QUAD == 4) {
    const ulonglong2* kp = reinterpret_cast<const ulonglong2*>(a.all_keys + (size_t)b * (size_t)(bw * bh) + p);
    const ulonglong2 k01 = __ldcs(kp), k23 = __ldcs(kp + 1);
    key[0] = k01.x; key[1] = k01.y; key[2] = k23.x; key[3] = k23.y;
  } else {
#pragma unroll
    for (int k = 0; k < SHADE_QUAD; ++k) key[k] = __ldcs(a.all_keys + (size_t)b * (size_t)(bw * bh) + p + k);
  }
  float L[3];
  normalise_light(a.light, L);
  int t[SHADE_QUAD], Px[SHADE_QUAD];
#pragma unroll
  for (int k = 0; k < SHADE_QUAD; ++k) {
    t[k] = (key[k] != CLEAR_KEY && x0 + k < g.W) ? (int)(unsigned)(key[k] & 0xFFFFFFFFu) : -1;
    Px[k] = 256 * (x0 + k) + 128;
  }
  float4 c[SHADE_QUAD];
  shade_batch<SHADE_QUAD>(a.verts, a.xv, a.M, a.idx, g.W, g.H, L, t, Px, 256 * y + 128, c);
  float dep[SHADE_QUAD];
  int prim[SHADE_QUAD];
#pragma unroll
  for (int k = 0; k < SHADE_QUAD; ++k) {
    dep[k] = t[k] >= 0 ? key_depth(key[k]) : 1.0f;
    prim[k] = t[k];
    if (t[k] >= 0 && a.sc.iters && !a.sc.forward) shader_sink(a.sc, shader_work(a.sc.iters, dep[k]));
  }
  const size_t o = (size_t)y * g.W + x0;
  if (SHADE_QUAD == 4 && x0 + SHADE_QUAD <= g.W && (o & 3) == 0) {
    float4* rp = reinterpret_cast<float4*>(a.out_rgba) + o;
#pragma unroll
    for (int k = 0; k < SHADE_QUAD; ++k) __stcs(rp + k, c[k]);
    __stcs(reinterpret_cast<float4*>(a.out_depth + o), make_float4(dep[0], dep[SHADE_QUAD > 1 ? 1 : 0], dep[SHADE_QUAD > 2 ? 2 : 0], dep[SHADE_QUAD > 3 ? 3 : 0]));
    __stcs(reinterpret_cast<int4*>(a.out_primid + o), make_int4(prim[0], prim[SHADE_QUAD > 1 ? 1 : 0], prim[SHADE_QUAD > 2 ? 2 : 0], prim[SHADE_QUAD > 3 ? 3 : 0]));
  } else {
#pragma unroll
    for (int k = 0; k < SHADE_QUAD; ++k) {
      if (x0 + k >= g.W) break;
      reinterpret_cast<float4*>(a.out_rgba)[o + k] = c[k];
      a.out_depth[o + k] = dep[k];
      a.out_primid[o + k] = prim[k];
    }
  }
}

// ---------------------------------------------------------------------------
// k_shade1: the deferred resolve with one pixel per thread (row-major, so the
// output stores are coalesced) and no per-pixel setup: the winner's
// orientation comes from its snapped corners' area sign alone (the O2 swap of
// corners 1 and 2), then the O7 arithmetic of shade_math in the same order.
// Pixels of bins without pairs (k_tile skipped them) and of overflowed frames
// are background without a key load.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float4 shade_lean(const float* __restrict__ verts, const int4* __restrict__ xv,
                                             const Mat4& M, const int32_t* __restrict__ idx, int W, int H,
                                             const float L[3], int t, int Px, int Py) {
  const int i0 = __ldg(idx + 3ll * t), i1 = __ldg(idx + 3ll * t + 1), i2 = __ldg(idx + 3ll * t + 2);
  int4 c0, c1, c2;
  if (xv) {
    c0 = __ldg(xv + i0); c1 = __ldg(xv + i1); c2 = __ldg(xv + i2);
  } else {
    const float4 p0 = load_pos(verts, i0), p1 = load_pos(verts, i1), p2 = load_pos(verts, i2);
    c0 = transform_vertex(p0, M, W, H);
    c1 = transform_vertex(p1, M, W, H);
    c2 = transform_vertex(p2, M, W, H);
  }
  float4 m0 = __ldg(reinterpret_cast<const float4*>(verts + 8ll * i0 + 4));
  float4 m1 = __ldg(reinterpret_cast<const float4*>(verts + 8ll * i1 + 4));
  float4 m2 = __ldg(reinterpret_cast<const float4*>(verts + 8ll * i2 + 4));
  long long area2 = (long long)(c1.x - c0.x) * (long long)(c2.y - c0.y) -
                    (long long)(c1.y - c0.y) * (long long)(c2.x - c0.x);
  if (area2 < 0) {  // O2 orientation normalisation (as setup_tri)
    const int4 ti = c1; c1 = c2; c2 = ti;
    const float4 tm = m1; m1 = m2; m2 = tm;
    area2 = -area2;
  }
  const float rw0 = __int_as_float(c0.w), rw1 = __int_as_float(c1.w), rw2 = __int_as_float(c2.w);
  const long long w0 = (long long)(c2.x - c1.x) * (Py - c1.y) - (long long)(c2.y - c1.y) * (Px - c1.x);
  const long long w1 = (long long)(c0.x - c2.x) * (Py - c2.y) - (long long)(c0.y - c2.y) * (Px - c2.x);
  const long long w2 = (long long)(c1.x - c0.x) * (Py - c0.y) - (long long)(c1.y - c0.y) * (Px - c0.x);
  const float inv = __frcp_rn(__ll2float_rn(area2));
  const float l0 = __fmul_rn(__fmul_rn(__ll2float_rn(w0), inv), rw0);
  const float l1 = __fmul_rn(__fmul_rn(__ll2float_rn(w1), inv), rw1);
  const float l2 = __fmul_rn(__fmul_rn(__ll2float_rn(w2), inv), rw2);
  const float vx = __fmaf_rn(l2, m2.x, __fmaf_rn(l1, m1.x, __fmul_rn(l0, m0.x)));
  const float vy = __fmaf_rn(l2, m2.y, __fmaf_rn(l1, m1.y, __fmul_rn(l0, m0.y)));
  const float vz = __fmaf_rn(l2, m2.z, __fmaf_rn(l1, m1.z, __fmul_rn(l0, m0.z)));
  const float d2 = __fmaf_rn(vx, vx, __fmaf_rn(vy, vy, __fmul_rn(vz, vz)));
  float lam = 0.0f;
  if (d2 != 0.0f) {
    const float q = __fdiv_rn(__fmaf_rn(vx, L[0], __fmaf_rn(vy, L[1], __fmul_rn(vz, L[2]))), __fsqrt_rn(d2));
    lam = (q > 0.0f) ? q : 0.0f;
  }
  return make_float4(__fmul_rn(0.80f, lam), __fmul_rn(0.75f, lam), __fmul_rn(0.65f, lam), 1.0f);
}

__global__ void __launch_bounds__(256) k_shade1(const __grid_constant__ ResolveArgs a) {
  pdl_wait();
  pdl_trigger();
  const Grid g = a.g;
  const long long o = (long long)blockIdx.x * 256 + threadIdx.x;
  if (o >= (long long)g.W * g.H) return;
  const int y = (int)(o / g.W), x = (int)(o % g.W);
  const int bw = 1 << g.bw_log2, bh = 1 << g.bh_log2;
  const int b = (y >> g.bh_log2) * g.binsX + (x >> g.bw_log2);
  const bool empty = a.bin_start == nullptr ? false
                     : (a.ctl->overflow_tag == a.ctl->frame + 1 || __ldg(a.bin_start + b + 1) == __ldg(a.bin_start + b));
  const u64 key = empty ? CLEAR_KEY
                        : __ldcs(a.all_keys + (size_t)b * (size_t)(bw * bh) + (y & (bh - 1)) * bw + (x & (bw - 1)));
  float4 c = make_float4(0.f, 0.f, 0.f, 0.f);
  float dep = 1.0f;
  int prim = -1;
  if (key != CLEAR_KEY) {
    float L[3];
    normalise_light(a.light, L);
    prim = (int)(unsigned)(key & 0xFFFFFFFFu);
    dep = key_depth(key);
    c = shade_lean(a.verts, a.xv, a.M, a.idx, g.W, g.H, L, prim, 256 * x + 128, 256 * y + 128);
    if (a.sc.iters && !a.sc.forward) shader_sink(a.sc, shader_work(a.sc.iters, dep));
  }
  __stcs(reinterpret_cast<float4*>(a.out_rgba) + o, c);
  __stcs(a.out_depth + o, dep);
  __stcs(a.out_primid + o, prim);
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
template <typename Kern, typename... Args>
static cudaError_t launch_ex(Kern kern, int grid, int threads, size_t smem, bool pdl,
                             cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

static int sm_count() {  // of the current device (contexts may live on different GPUs)
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 148;
}

cudaError_t launch_vertex(const VertexArgs& a, bool pdl, cudaStream_t s) {
  // known count: one thread per vertex; unknown (device-side count): persistent
  const long long want = a.n_verts >= 0 ? (a.n_verts + VX_VPT * VX_THREADS - 1) / (VX_VPT * VX_THREADS) : 8ll * sm_count();
  return launch_ex(k_vertex, (int)(want > 0 ? want : 1), VX_THREADS, 0, pdl, s, a);
}

cudaError_t launch_index_max(const int32_t* idx, long long n, Control* ctl, bool pdl, cudaStream_t s) {
  // a few int4 loads in flight per thread: about 2 waves of CTAs
#ifndef PIKO_IMAX_CTAS_PER_SM
#define PIKO_IMAX_CTAS_PER_SM 4
#endif
  const long long want = std::min<long long>((n / 4 + 255) / 256, (long long)PIKO_IMAX_CTAS_PER_SM * sm_count());
  return launch_ex(k_index_max, (int)(want > 0 ? want : 1), 256, 0, pdl, s, idx, n, ctl);
}
cudaError_t launch_setup(const SetupArgs& a, int grid, bool pdl, cudaStream_t s) {
  // the chunk-list arrays (the tail of K1Smem from bm on) only in chunk-list
  // frames: otherwise the smaller carve-out leaves the L1 to the corner gathers
  // (set per launch: the attribute belongs to the current device's context)
  const size_t smem = a.cl_ent ? sizeof(K1Smem) : offsetof(K1Smem, bigg);
  cudaError_t e = a.xv ? cudaFuncSetAttribute(k_setup<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                       : cudaFuncSetAttribute(k_setup<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (!a.xv) return launch_ex(k_setup<true>, grid, K1_THREADS, smem, pdl, s, a);
  return launch_ex(k_setup<false>, grid, K1_THREADS, smem, pdl, s, a);
}
cudaError_t launch_radix_pass(const RadixArgs& a, int grid, bool pdl, cudaStream_t s) {
  if (a.expand) {
    const size_t smem = sizeof(RadixSmem) + sizeof(ExpandSmem);
    cudaError_t e = cudaFuncSetAttribute(k_radix_pass<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    return launch_ex(k_radix_pass<true>, grid, RX_THREADS, smem, pdl, s, a);
  }
  const size_t smem = sizeof(RadixSmem);
  cudaError_t e = cudaFuncSetAttribute(k_radix_pass<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_ex(k_radix_pass<false>, grid, RX_THREADS, smem, pdl, s, a);
}
cudaError_t launch_bin_scan(const RadixArgs& a, int grid, bool pdl, cudaStream_t s) {
  return launch_ex(k_bin_scan, grid, SCAN_THREADS, 0, pdl, s, a);
}
cudaError_t launch_dice_rate(const DiceArgs& a, cudaStream_t s) {
  k_dice_rate<<<1, 1024, 0, s>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_dice(const DiceArgs& a, cudaStream_t s) {
  if (a.n > 0) k_dice<<<(unsigned)a.n, 256, 0, s>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_cm_scan(const CmArgs& a, int grid, bool pdl, cudaStream_t s) {
  return launch_ex(k_cm_scan, grid, 256, 0, pdl, s, a);
}
cudaError_t launch_cm_scatter(const CmArgs& a, int grid, bool pdl, cudaStream_t s) {
  const size_t smem = sizeof(CmSmem);
  cudaError_t e = cudaFuncSetAttribute(k_cm_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_ex(k_cm_scatter, grid, CM_THREADS, smem, pdl, s, a);
}
cudaError_t launch_cl_bins(const ClArgs& a, int grid, bool pdl, cudaStream_t s) {
  const size_t smem = sizeof(ClbSmem);
  cudaError_t e = cudaFuncSetAttribute(k_cl_bins, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_ex(k_cl_bins, grid, CLB_THREADS, smem, pdl, s, a);
}

#endif  // PIKO_TILE_TU

// k_tile instantiations (16 bin shapes x coverage x keys-only): with
// -DPIKO_SPLIT_TILES they are compiled in four extra translation units
// (-DPIKO_TILE_TU=8/16/32/64, one per bin width) in parallel with this one.
#if !defined(PIKO_SPLIT_TILES) || defined(PIKO_TILE_TU)
template <int BW, int BH>
static TileKernel tile_kernel_t(bool cov, bool keys_only) {
  constexpr int NPX = BW * BH;
  constexpr int THREADS = NPX < TILE_THREADS ? NPX : TILE_THREADS;
  TileKernel k;
  k.threads = THREADS;
  k.smem = sizeof(TileSmem<BW, BH, THREADS>) + (cov ? (size_t)NPX * 4 : 0);
  if (keys_only) k.fn = cov ? k_tile<BW, BH, THREADS, true, true> : k_tile<BW, BH, THREADS, false, true>;
  else k.fn = cov ? k_tile<BW, BH, THREADS, true, false> : k_tile<BW, BH, THREADS, false, false>;
  return k;
}
#define PIKO_TILE_BW(W_)                                                              \
  TileKernel tile_kernel_bw##W_(int bh, bool cov, bool keys_only) {                   \
    if (bh == 8) return tile_kernel_t<W_, 8>(cov, keys_only);                        \
    if (bh == 16) return tile_kernel_t<W_, 16>(cov, keys_only);                      \
    if (bh == 32) return tile_kernel_t<W_, 32>(cov, keys_only);                      \
    if (bh == 64) return tile_kernel_t<W_, 64>(cov, keys_only);                      \
    return TileKernel{};                                                              \
  }
#if !defined(PIKO_TILE_TU) || PIKO_TILE_TU == 8
PIKO_TILE_BW(8)
#endif
#if !defined(PIKO_TILE_TU) || PIKO_TILE_TU == 16
PIKO_TILE_BW(16)
#endif
#if !defined(PIKO_TILE_TU) || PIKO_TILE_TU == 32
PIKO_TILE_BW(32)
#endif
#if !defined(PIKO_TILE_TU) || PIKO_TILE_TU == 64
PIKO_TILE_BW(64)
#endif
#endif

#ifndef PIKO_TILE_TU
static TileKernel tile_kernel(int bw, int bh, bool cov, bool keys_only) {
  switch (bw) {
    case 8: return tile_kernel_bw8(bh, cov, keys_only);
    case 16: return tile_kernel_bw16(bh, cov, keys_only);
    case 32: return tile_kernel_bw32(bh, cov, keys_only);
    case 64: return tile_kernel_bw64(bh, cov, keys_only);
  }
  return TileKernel{};
}

cudaError_t launch_tile(const TileArgs& a, int bw, int bh, int grid, bool cov, bool keys_only,
                        bool pdl, cudaStream_t s) {
  const TileKernel k = tile_kernel(bw, bh, cov, keys_only);
  if (!k.fn) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k.smem);
  if (e != cudaSuccess) return e;
  return launch_ex(k.fn, grid, k.threads, k.smem, pdl, s, a);
}

// persistent grid: all CTAs resident at once (the queue needs no more)
int tile_grid(int bw, int bh, bool cov, bool keys_only) {
  const TileKernel k = tile_kernel(bw, bh, cov, keys_only);
  int dev = 0, sms = 148, occ = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (k.fn) {
    cudaFuncSetAttribute(k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k.smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k.fn, k.threads, k.smem);
  }
  return sms * (occ > 0 ? occ : 1);
}

cudaError_t launch_freepipe(const FreePipeArgs& a, bool pdl, cudaStream_t s) {
  const long long grid = (a.n_tris + 1023) / 1024;
  return launch_ex(k_freepipe, (int)(grid > 0 ? grid : 1), 256, 0, pdl, s, a);
}
cudaError_t launch_fp_resolve(const FreePipeArgs& a, bool pdl, cudaStream_t s) {
  const long long grid = ((long long)a.W * a.H + 255) / 256;
  return launch_ex(k_fp_resolve, (int)grid, 256, 0, pdl, s, a);
}

// Baseline stages: 0 raster, 1 fragment shader, 2 depth test, 3 composite
// (winners), 4 composite (background + depth-buffer clear)
cudaError_t launch_baseline(const BaselineArgs& a, int stage, bool pdl, cudaStream_t s) {
  const long long npx = (long long)a.W * a.H;
  const int frag_grid = 16 * sm_count();  // grid-stride over the device-side count
  switch (stage) {
    case 0: return launch_ex(k_bl_raster, (int)std::max<long long>((a.n_tris + 255) / 256, 1), 256, 0, pdl, s, a);
    case 1: return launch_ex(k_bl_fs, frag_grid, 256, 0, pdl, s, a);
    case 2: return launch_ex(k_bl_depth, frag_grid, 256, 0, pdl, s, a);
    case 3: return launch_ex(k_bl_composite, frag_grid, 256, 0, pdl, s, a);
    case 4: return launch_ex(k_bl_clear, (int)((npx + 255) / 256), 256, 0, pdl, s, a);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_shade(const ResolveArgs& a, bool pdl, cudaStream_t s) {
  if (a.bin_start) {  // one pixel per thread, empty bins known from the CSR (k_tile skipped them)
    const long long n = (long long)a.g.W * a.g.H;
    return launch_ex(k_shade1, (int)((n + 255) / 256), 256, 0, pdl, s, a);
  }
  const long long nq = (long long)((a.g.W + SHADE_QUAD - 1) / SHADE_QUAD) * a.g.H;
  return launch_ex(k_shade, (int)((nq + 255) / 256), 256, 0, pdl, s, a);
}
cudaError_t launch_resolve(const ResolveArgs& a, bool pdl, cudaStream_t s) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((a.g.W + 31) / 32, (a.g.H + 7) / 8);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k_resolve, a);
}

#endif  // PIKO_TILE_TU

}  // namespace piko
