// kernels.cu -- the hot path of the binned rasterizer, hand-written for sm_100a.
//
//   k_setup      vertex transform + fixed-point setup + AssignBin count, fused
//                with a decoupled-look-back exclusive scan of the per-triangle
//                pair counts and the expansion of (bin, primID) pairs in
//                primitive order.
//   k_bin_scan   exclusive scan of the per-bin pair counts -> CSR bin_start, plus
//                the digit histograms of the stable LSD radix passes.
//   k_radix_pass one stable LSD pass (8-bit digit) of the pairs by bin id:
//                warp match-any ranking, per-digit decoupled look-back,
//                shared-memory staged scatter.  After the last pass the values
//                are the CSR bin_prims, ascending primID within each bin.
//   k_tile       Process, one CTA per owned bin (LoadBalance):
//                tile z-buffer of packed 64-bit (depth, primID) keys in shared
//                memory, triangle-parallel raster for small triangles and
//                pixel-parallel raster for large ones, then per-pixel Lambert
//                shade (Listing 1) and a vectorised write-back.
//   k_resolve    multi-GPU rank 0: shade gathered tile keys into the frame.
//
// Arithmetic follows DESIGN.md R1..R18 with a pinned float op order (IEEE
// round-to-nearest intrinsics, explicit fma); this TU is compiled with
// --fmad=false so no other contraction can happen.
#include <cstdint>

#include "piko_internal.h"

namespace piko {

constexpr unsigned long long CLEAR_KEY = 0xFFFFFFFFFFFFFFFFull;
constexpr float W_EPS = 1e-6f;
constexpr float GUARD = 4194304.0f;  // 2^22 subpixels

// ---------------------------------------------------------------------------
// memory-model helpers for the look-back scans
// ---------------------------------------------------------------------------
__device__ __forceinline__ void st_release64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed32(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_relaxed32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

constexpr unsigned long long LB_AGG = 1ull << 62;   // aggregate published
constexpr unsigned long long LB_INC = 2ull << 62;   // inclusive prefix published
constexpr unsigned long long LB_VAL = (1ull << 62) - 1;

// Decoupled look-back (one full warp): publish this chunk's aggregate, sum the
// predecessors' values back to the nearest inclusive prefix (32 at a time),
// publish the inclusive prefix.  Returns the exclusive prefix.
__device__ unsigned long long lookback_warp(unsigned long long* status, unsigned chunk,
                                            unsigned long long agg, int lane) {
  if (lane == 0) st_release64(&status[chunk], (chunk == 0 ? LB_INC : LB_AGG) | agg);
  if (chunk == 0) return 0;
  unsigned long long excl = 0;
  long long hi = (long long)chunk - 1;
  for (;;) {
    long long i = hi - lane;
    unsigned long long s = (i >= 0) ? ld_acquire64(&status[i]) : LB_INC;
    unsigned flag = (unsigned)(s >> 62);
    unsigned inc = __ballot_sync(0xffffffffu, flag == 2u);
    unsigned notready = __ballot_sync(0xffffffffu, flag == 0u);
    int k = inc ? (__ffs(inc) - 1) : 32;
    unsigned need = (k >= 31) ? 0xffffffffu : ((2u << k) - 1u);
    if (notready & need) continue;  // a predecessor has not published yet
    unsigned long long v = (lane <= k) ? (s & LB_VAL) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    excl += v;
    if (k < 32) break;
    hi -= 32;
  }
  if (lane == 0) st_release64(&status[chunk], LB_INC | (excl + agg));
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

__device__ __forceinline__ bool xform_corner(const float* __restrict__ verts, int vid,
                                             const Mat4& M, float hw, float hh, int& X,
                                             int& Y, float& zw, float& rw) {
  const float4 p = __ldg(reinterpret_cast<const float4*>(verts + 8ll * vid));
  const float cx = __fmaf_rn(M.m[0], p.x, __fmaf_rn(M.m[1], p.y, __fmaf_rn(M.m[2], p.z, M.m[3])));
  const float cy = __fmaf_rn(M.m[4], p.x, __fmaf_rn(M.m[5], p.y, __fmaf_rn(M.m[6], p.z, M.m[7])));
  const float cz = __fmaf_rn(M.m[8], p.x, __fmaf_rn(M.m[9], p.y, __fmaf_rn(M.m[10], p.z, M.m[11])));
  const float cw = __fmaf_rn(M.m[12], p.x, __fmaf_rn(M.m[13], p.y, __fmaf_rn(M.m[14], p.z, M.m[15])));
  if (!(isfinite(cx) && isfinite(cy) && isfinite(cz) && isfinite(cw))) return false;
  if (!(cw > W_EPS)) return false;
  const float r = __fdiv_rn(1.0f, cw);
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

// Full setup of triangle with corner vertex ids (i0,i1,i2); false = culled.
__device__ __forceinline__ bool setup_tri(const float* __restrict__ verts, int i0, int i1, int i2,
                                          const Mat4& M, int W, int H, Tri& o) {
  const float hw = __fmul_rn(0.5f, __int2float_rn(W));
  const float hh = __fmul_rn(0.5f, __int2float_rn(H));
  bool ok = xform_corner(verts, i0, M, hw, hh, o.X0, o.Y0, o.zw0, o.rw0);
  ok = ok && xform_corner(verts, i1, M, hw, hh, o.X1, o.Y1, o.zw1, o.rw1);
  ok = ok && xform_corner(verts, i2, M, hw, hh, o.X2, o.Y2, o.zw2, o.rw2);
  if (!ok) return false;
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
__device__ __forceinline__ unsigned owned_in_rect(int tx0, int ty0, int tx1, int ty1, const Grid& g) {
  if (g.nranks == 1) return (unsigned)((tx1 - tx0 + 1) * (ty1 - ty0 + 1));
  unsigned n = 0;
  for (int ty = ty0; ty <= ty1; ++ty) {
    const int base = ty * g.binsX + tx0;  // bin of tx0 in this row
    int first = (g.rank - base % g.nranks + g.nranks) % g.nranks;  // offset of 1st owned
    const int w = tx1 - tx0 + 1;
    if (first < w) n += (unsigned)((w - 1 - first) / g.nranks + 1);
  }
  return n;
}

// ---------------------------------------------------------------------------
// K1: vertex + setup + count + chunk scan + pair expansion (persistent CTAs)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(K1_THREADS) k_setup(SetupArgs a) {
  __shared__ unsigned s_chunk;
  __shared__ unsigned long long s_warp[K1_THREADS / 32];
  __shared__ unsigned long long s_base;
  __shared__ unsigned s_live;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Grid g = a.g;

  for (;;) {
    if (tid == 0) { s_chunk = atomicAdd(&a.ctl->ticket_k1, 1u); s_live = 0; }
    __syncthreads();
    const unsigned chunk = s_chunk;
    const long long t0 = (long long)chunk * K1_CHUNK;
    if (t0 >= a.n_tris) break;  // uniform across the CTA

    // ---- setup of this thread's 4 consecutive triangles -------------------
    const long long tb = t0 + (long long)tid * K1_TPT;
    int vi[12];
    if (tb + K1_TPT <= a.n_tris) {
      const int4* p = reinterpret_cast<const int4*>(a.idx + 3 * tb);
      const int4 q0 = __ldg(p), q1 = __ldg(p + 1), q2 = __ldg(p + 2);
      vi[0] = q0.x; vi[1] = q0.y; vi[2] = q0.z; vi[3] = q0.w;
      vi[4] = q1.x; vi[5] = q1.y; vi[6] = q1.z; vi[7] = q1.w;
      vi[8] = q2.x; vi[9] = q2.y; vi[10] = q2.z; vi[11] = q2.w;
    } else {
#pragma unroll
      for (int k = 0; k < 12; ++k)
        vi[k] = (tb + k / 3 < a.n_tris) ? __ldg(a.idx + 3 * tb + k) : 0;
    }
    unsigned cnt[K1_TPT];
    int rect[K1_TPT];  // packed tile rect: tx0 | ty0<<8 ... stored as 4 x 8 bit? use 2 ints
    int rect2[K1_TPT];
    unsigned live = 0;
#pragma unroll
    for (int k = 0; k < K1_TPT; ++k) {
      cnt[k] = 0; rect[k] = 0; rect2[k] = 0;
      const long long t = tb + k;
      if (t >= a.n_tris) continue;
      Tri o;
      if (!setup_tri(a.verts, vi[3 * k], vi[3 * k + 1], vi[3 * k + 2], a.M, g.W, g.H, o)) continue;
      const int tx0 = o.px0 >> g.bw_log2, tx1 = o.px1 >> g.bw_log2;
      const int ty0 = o.py0 >> g.bh_log2, ty1 = o.py1 >> g.bh_log2;
      const unsigned c = owned_in_rect(tx0, ty0, tx1, ty1, g);
      if (c == 0) continue;
      cnt[k] = c;
      rect[k] = tx0 | (ty0 << 16);
      rect2[k] = tx1 | (ty1 << 16);
      ++live;
      // depth plane (O6) through the snapped corners
      const float dx1 = __int2float_rn(o.X1 - o.X0), dy1 = __int2float_rn(o.Y1 - o.Y0);
      const float dx2 = __int2float_rn(o.X2 - o.X0), dy2 = __int2float_rn(o.Y2 - o.Y0);
      const float dz1 = __fsub_rn(o.zw1, o.zw0), dz2 = __fsub_rn(o.zw2, o.zw0);
      const float inv = __fdiv_rn(1.0f, __ll2float_rn(o.area2));
      const float za = __fmul_rn(__fmaf_rn(dz1, dy2, -__fmul_rn(dz2, dy1)), inv);
      const float zb = __fmul_rn(__fmaf_rn(dz2, dx1, -__fmul_rn(dz1, dx2)), inv);
      int4* r = a.rec + 3 * t;
      r[0] = make_int4(o.X0, o.Y0, o.X1, o.Y1);
      r[1] = make_int4(o.X2, o.Y2, __float_as_int(o.zw0), __float_as_int(za));
      r[2] = make_int4(__float_as_int(zb), o.px0 | (o.py0 << 16), o.px1 | (o.py1 << 16),
                       o.small ? REC_SMALL : 0);
    }

    // ---- CTA exclusive scan of the pair counts ----------------------------
    const unsigned long long mine = (unsigned long long)cnt[0] + cnt[1] + cnt[2] + cnt[3];
    unsigned long long inc = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long v = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += v;
    }
    if (lane == 31) s_warp[warp] = inc;
    if (live) atomicAdd(&s_live, live);
    __syncthreads();
    unsigned long long wbase = 0, total = 0;
#pragma unroll
    for (int w = 0; w < K1_THREADS / 32; ++w) {
      const unsigned long long v = s_warp[w];
      wbase += (w < warp) ? v : 0ull;
      total += v;
    }
    if (warp == 0) {
      const unsigned long long ex = lookback_warp(a.status, chunk, total, lane);
      if (lane == 0) {
        s_base = ex;
        if (s_live) atomicAdd(&a.ctl->n_live, (unsigned long long)s_live);
        if (t0 + K1_CHUNK >= a.n_tris) a.ctl->n_pairs = ex + total;  // last chunk
      }
    }
    __syncthreads();

    // ---- expansion: pairs (bin, t) in primitive order ----------------------
    unsigned long long off = s_base + wbase + (inc - mine);
    if (off + mine > a.cap) {
      if (mine) atomicOr(&a.ctl->overflow, 1u);
    } else {
#pragma unroll
      for (int k = 0; k < K1_TPT; ++k) {
        if (!cnt[k]) continue;
        const int t = (int)(tb + k);
        const int tx0 = rect[k] & 0xffff, ty0 = rect[k] >> 16;
        const int tx1 = rect2[k] & 0xffff, ty1 = rect2[k] >> 16;
        for (int ty = ty0; ty <= ty1; ++ty) {
          for (int tx = tx0; tx <= tx1; ++tx) {
            const int b = ty * g.binsX + tx;
            if (g.nranks > 1 && (b % g.nranks) != g.rank) continue;
            a.pair_keys[off] = (uint32_t)b;
            a.pair_vals[off] = t;
            atomicAdd(&a.bin_count[b], 1u);
            ++off;
          }
        }
      }
    }
    __syncthreads();  // s_chunk / s_base reuse
  }
}

// ---------------------------------------------------------------------------
// K2: bin counts -> CSR bin_start (decoupled look-back), digit histograms
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(SCAN_THREADS) k_bin_scan(ScanArgs a) {
  __shared__ unsigned s_chunk;
  __shared__ unsigned long long s_warp[SCAN_THREADS / 32];
  __shared__ unsigned long long s_base;
  __shared__ unsigned s_hist[MAX_PASSES][RX_RADIX];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < MAX_PASSES * RX_RADIX; i += SCAN_THREADS) (&s_hist[0][0])[i] = 0;
  const bool ovf = a.ctl->overflow != 0;
  for (;;) {
    if (tid == 0) s_chunk = atomicAdd(&a.ctl->ticket_scan, 1u);
    __syncthreads();
    const unsigned chunk = s_chunk;
    const long long b0 = (long long)chunk * SCAN_CHUNK;
    if (b0 >= a.NB) break;
    const long long bt = b0 + (long long)tid * SCAN_ITEMS;
    unsigned c[SCAN_ITEMS];
    unsigned long long mine = 0;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) {
      const long long b = bt + k;
      c[k] = (b < a.NB && !ovf) ? a.bin_count[b] : 0u;
      mine += c[k];
      if (c[k]) {
        for (int p = 0; p < a.npass; ++p)
          atomicAdd(&s_hist[p][(b >> (RX_BITS * p)) & (RX_RADIX - 1)], c[k]);
      }
    }
    unsigned long long inc = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long v = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += v;
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    unsigned long long wbase = 0, total = 0;
#pragma unroll
    for (int w = 0; w < SCAN_THREADS / 32; ++w) {
      const unsigned long long v = s_warp[w];
      wbase += (w < warp) ? v : 0ull;
      total += v;
    }
    if (warp == 0) {
      const unsigned long long ex = lookback_warp(a.status, chunk, total, lane);
      if (lane == 0) s_base = ex;
    }
    __syncthreads();
    unsigned long long run = s_base + wbase + (inc - mine);
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) {
      const long long b = bt + k;
      if (b < a.NB) {
        a.bin_start[b] = (int32_t)run;
        a.bin_count[b] = 0u;  // ready for the next frame
      }
      run += c[k];
    }
    if (b0 + SCAN_CHUNK >= a.NB && tid == SCAN_THREADS - 1) a.bin_start[a.NB] = (int32_t)run;
    __syncthreads();
  }
  __syncthreads();
  for (int i = tid; i < a.npass * RX_RADIX; i += SCAN_THREADS) {
    const unsigned v = (&s_hist[0][0])[i];
    if (v) atomicAdd(&a.ctl->digit_hist[0][0] + i, v);
  }
}

// ---------------------------------------------------------------------------
// K3: one stable LSD radix pass over the (bin, primID) pairs
// ---------------------------------------------------------------------------
constexpr unsigned RX_AGG = 1u << 30, RX_INC = 2u << 30, RX_VAL = (1u << 30) - 1;

__global__ void __launch_bounds__(RX_THREADS) k_radix_pass(RadixArgs a) {
  __shared__ unsigned s_whist[RX_WARPS][RX_RADIX];
  __shared__ unsigned s_keys[RX_CHUNK];
  __shared__ int s_vals[RX_CHUNK];
  __shared__ unsigned s_prefix[RX_RADIX];
  __shared__ unsigned s_lstart[RX_RADIX];
  __shared__ unsigned s_gstart[RX_RADIX];
  __shared__ unsigned s_wsum[RX_WARPS];
  __shared__ unsigned s_chunk;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lanemask_lt = (1u << lane) - 1u;
  if (a.ctl->overflow) return;
  const unsigned long long P = a.ctl->n_pairs;

  // block exclusive scan of 256 values (one per thread)
  auto block_excl = [&](unsigned v) -> unsigned {
    unsigned inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) s_wsum[warp] = inc;
    __syncthreads();
    unsigned base = 0;
    for (int w = 0; w < warp; ++w) base += s_wsum[w];
    __syncthreads();
    return base + inc - v;
  };
  s_prefix[tid] = block_excl(a.ctl->digit_hist[a.pass][tid]);

  for (;;) {
    if (tid == 0) s_chunk = atomicAdd(&a.ctl->ticket_rx[a.pass], 1u);
#pragma unroll
    for (int w = 0; w < RX_WARPS; ++w) s_whist[w][tid] = 0;
    __syncthreads();
    const unsigned chunk = s_chunk;
    const unsigned long long c0 = (unsigned long long)chunk * RX_CHUNK;
    if (c0 >= P) break;

    unsigned key[RX_ITEMS];
    int val[RX_ITEMS];
    unsigned rank[RX_ITEMS];
    const unsigned long long wb = c0 + (unsigned long long)warp * (RX_ITEMS * 32) + lane;
#pragma unroll
    for (int j = 0; j < RX_ITEMS; ++j) {
      const unsigned long long pos = wb + j * 32;
      const bool valid = pos < P;
      key[j] = valid ? a.keys_in[pos] : 0u;
      val[j] = valid ? a.vals_in[pos] : 0;
    }
#pragma unroll
    for (int j = 0; j < RX_ITEMS; ++j) {
      const unsigned long long pos = wb + j * 32;
      const bool valid = pos < P;
      const unsigned d = valid ? ((key[j] >> a.shift) & (RX_RADIX - 1)) : RX_RADIX;
      const unsigned peers = __match_any_sync(0xffffffffu, d);
      unsigned prev = 0;
      if (valid) prev = s_whist[warp][d];
      __syncwarp();
      if (valid && lane == __ffs(peers) - 1) s_whist[warp][d] = prev + __popc(peers);
      __syncwarp();
      rank[j] = prev + __popc(peers & lanemask_lt);
    }
    __syncthreads();
    // per digit d = tid: exclusive offsets over warps, chunk total
    unsigned tot = 0;
#pragma unroll
    for (int w = 0; w < RX_WARPS; ++w) {
      const unsigned c = s_whist[w][tid];
      s_whist[w][tid] = tot;
      tot += c;
    }
    const unsigned lstart = block_excl(tot);
    s_lstart[tid] = lstart;
    // decoupled look-back per digit (thread tid owns digit tid)
    unsigned* st = a.status + (size_t)chunk * RX_RADIX + tid;
    unsigned excl = 0;
    if (chunk == 0) {
      st_relaxed32(st, RX_INC | tot);
    } else {
      st_relaxed32(st, RX_AGG | tot);
      const unsigned* q = st - RX_RADIX;
      for (;;) {
        unsigned s;
        do { s = ld_relaxed32(q); } while ((s >> 30) == 0u);
        excl += s & RX_VAL;
        if ((s >> 30) == 2u) break;
        q -= RX_RADIX;
      }
      st_relaxed32(st, RX_INC | (excl + tot));
    }
    s_gstart[tid] = s_prefix[tid] + excl;
    __syncthreads();
    // stage the chunk sorted by digit in shared memory
#pragma unroll
    for (int j = 0; j < RX_ITEMS; ++j) {
      const unsigned long long pos = wb + j * 32;
      if (pos < P) {
        const unsigned d = (key[j] >> a.shift) & (RX_RADIX - 1);
        const unsigned lp = s_lstart[d] + s_whist[warp][d] + rank[j];
        s_keys[lp] = key[j];
        s_vals[lp] = val[j];
      }
    }
    __syncthreads();
    const unsigned n = (unsigned)min((unsigned long long)RX_CHUNK, P - c0);
    for (unsigned i = tid; i < n; i += RX_THREADS) {
      const unsigned k = s_keys[i];
      const unsigned d = (k >> a.shift) & (RX_RADIX - 1);
      const unsigned g = s_gstart[d] + (i - s_lstart[d]);
      if (a.keys_out) a.keys_out[g] = k;
      a.vals_out[g] = s_vals[i];
    }
    __syncthreads();
  }
}

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
// bbox when r.small).  Returns the packed key or CLEAR_KEY; *covered for stats.
__device__ __forceinline__ unsigned long long eval_key(const RecView& r, int Px, int Py, int t,
                                                       bool& covered) {
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
  return ((unsigned long long)(__float_as_uint(z) & 0x7FFFFFFFu) << 32) | (unsigned)t;
}

// O7 shade of pixel sample (Px, Py) by triangle t (recomputes setup).
__device__ __forceinline__ float4 shade(const float* __restrict__ verts, const int32_t* __restrict__ idx,
                                        const Mat4& M, int W, int H, const float L[3], int t,
                                        int Px, int Py) {
  Tri o;
  const int i0 = __ldg(idx + 3ll * t), i1 = __ldg(idx + 3ll * t + 1), i2 = __ldg(idx + 3ll * t + 2);
  setup_tri(verts, i0, i1, i2, M, W, H, o);  // live: t won a pixel
  const long long w0 = (long long)(o.X2 - o.X1) * (Py - o.Y1) - (long long)(o.Y2 - o.Y1) * (Px - o.X1);
  const long long w1 = (long long)(o.X0 - o.X2) * (Py - o.Y2) - (long long)(o.Y0 - o.Y2) * (Px - o.X2);
  const long long w2 = (long long)(o.X1 - o.X0) * (Py - o.Y0) - (long long)(o.Y1 - o.Y0) * (Px - o.X0);
  const float inv = __fdiv_rn(1.0f, __ll2float_rn(o.area2));
  const float l0 = __fmul_rn(__fmul_rn(__ll2float_rn(w0), inv), o.rw0);
  const float l1 = __fmul_rn(__fmul_rn(__ll2float_rn(w1), inv), o.rw1);
  const float l2 = __fmul_rn(__fmul_rn(__ll2float_rn(w2), inv), o.rw2);
  const float4 n0 = __ldg(reinterpret_cast<const float4*>(verts + 8ll * o.v0 + 4));
  const float4 n1 = __ldg(reinterpret_cast<const float4*>(verts + 8ll * o.v1 + 4));
  const float4 n2 = __ldg(reinterpret_cast<const float4*>(verts + 8ll * o.v2 + 4));
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

__device__ __forceinline__ void normalise_light(const float in[3], float L[3]) {
  const float s = __fsqrt_rn(__fmaf_rn(in[0], in[0], __fmaf_rn(in[1], in[1], __fmul_rn(in[2], in[2]))));
  L[0] = __fdiv_rn(in[0], s);
  L[1] = __fdiv_rn(in[1], s);
  L[2] = __fdiv_rn(in[2], s);
}

constexpr int SMALL_AREA = 16;  // clipped pixel-rect area handled by one thread

template <int BW, int BH, int THREADS, bool COV, bool KEYS_ONLY>
__global__ void __launch_bounds__(THREADS) k_tile(TileArgs a) {
  constexpr int NPX = BW * BH;
  constexpr int PPT = (NPX + THREADS - 1) / THREADS;
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned long long* s_key = reinterpret_cast<unsigned long long*>(smem);   // [NPX]
  int4* s_q = reinterpret_cast<int4*>(s_key + NPX);                          // [THREADS][3]
  int* s_qt = reinterpret_cast<int*>(s_q + 3 * THREADS);                     // [THREADS]
  unsigned* s_cov = reinterpret_cast<unsigned*>(s_qt + THREADS);             // [NPX] (COV)
  __shared__ int s_qn;

  const int tid = threadIdx.x;
  const Grid g = a.g;
  const int b = g.rank + blockIdx.x * g.nranks;  // owned bin (DirectMap across ranks)
  const int bx = b % g.binsX, by = b / g.binsX;
  const int x0 = bx * BW, y0 = by * BH;
  const int x1 = min(x0 + BW, g.W) - 1, y1 = min(y0 + BH, g.H) - 1;
  const bool ovf = a.ctl->overflow != 0;

#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    const int p = tid + k * THREADS;
    if (p < NPX) {
      s_key[p] = CLEAR_KEY;
      if (COV) s_cov[p] = 0;
    }
  }
  if (tid == 0) s_qn = 0;
  __syncthreads();

  const int s = ovf ? 0 : a.bin_start[b];
  const int e = ovf ? 0 : a.bin_start[b + 1];
  for (int base = s; base < e; base += THREADS) {
    const int i = base + tid;
    if (i < e) {
      const int t = a.bin_prims[i];
      const int4* rp = a.rec + 3ll * t;
      const int4 q0 = __ldg(rp), q1 = __ldg(rp + 1), q2 = __ldg(rp + 2);
      const RecView r = unpack(q0, q1, q2);
      const int rx0 = max(r.px0, x0), rx1 = min(r.px1, x1);
      const int ry0 = max(r.py0, y0), ry1 = min(r.py1, y1);
      const int area = (rx1 - rx0 + 1) * (ry1 - ry0 + 1);
      if (area <= SMALL_AREA) {
        for (int y = ry0; y <= ry1; ++y) {
          const int Py = 256 * y + 128;
          for (int x = rx0; x <= rx1; ++x) {
            bool cov;
            const unsigned long long key = eval_key(r, 256 * x + 128, Py, t, cov);
            const int p = (y - y0) * BW + (x - x0);
            if (COV && cov) atomicAdd(&s_cov[p], 1u);
            if (key != CLEAR_KEY) atomicMin(&s_key[p], key);
          }
        }
      } else {
        const int slot = atomicAdd(&s_qn, 1);
        s_q[3 * slot] = q0; s_q[3 * slot + 1] = q1; s_q[3 * slot + 2] = q2;
        s_qt[slot] = t;
      }
    }
    __syncthreads();
    const int n = s_qn;
    for (int k = 0; k < n; ++k) {
      const RecView r = unpack(s_q[3 * k], s_q[3 * k + 1], s_q[3 * k + 2]);
      const int t = s_qt[k];
#pragma unroll
      for (int j = 0; j < PPT; ++j) {
        const int p = tid + j * THREADS;
        if (p >= NPX) continue;
        const int x = x0 + (p % BW), y = y0 + (p / BW);
        if (x < r.px0 || x > r.px1 || y < r.py0 || y > r.py1) continue;
        bool cov;
        const unsigned long long key = eval_key(r, 256 * x + 128, 256 * y + 128, t, cov);
        if (COV && cov) s_cov[p] += 1u;
        if (key < s_key[p]) s_key[p] = key;
      }
    }
    __syncthreads();
    if (tid == 0) s_qn = 0;
    __syncthreads();
  }

  // ---- write-back ------------------------------------------------------------
  if (KEYS_ONLY) {
    unsigned long long* dst = a.tile_keys + (size_t)blockIdx.x * NPX;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      const int p = tid + k * THREADS;
      if (p < NPX) dst[p] = s_key[p];
    }
    return;
  }
  float L[3];
  normalise_light(a.light, L);
#pragma unroll
  for (int k = 0; k < PPT; ++k) {
    const int p = tid + k * THREADS;
    if (p >= NPX) continue;
    const int x = x0 + (p % BW), y = y0 + (p / BW);
    if (x > x1 || y > y1) continue;
    const unsigned long long key = s_key[p];
    const size_t o = (size_t)y * g.W + x;
    float4 c = make_float4(0.f, 0.f, 0.f, 0.f);
    float depth = 1.0f;
    int prim = -1;
    if (key != CLEAR_KEY) {
      prim = (int)(unsigned)(key & 0xFFFFFFFFu);
      depth = __uint_as_float((unsigned)(key >> 32));
      c = shade(a.verts, a.idx, a.M, g.W, g.H, L, prim, 256 * x + 128, 256 * y + 128);
    }
    reinterpret_cast<float4*>(a.out_rgba)[o] = c;
    a.out_depth[o] = depth;
    a.out_primid[o] = prim;
    if (COV) a.out_cov[o] = s_cov[p];
  }
}

// ---------------------------------------------------------------------------
// K7 (multi-GPU rank 0): resolve gathered tile keys -> shaded frame
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_resolve(ResolveArgs a) {
  const Grid g = a.g;
  const int x = blockIdx.x * 32 + (threadIdx.x & 31);
  const int y = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (x >= g.W || y >= g.H) return;
  const int bw = 1 << g.bw_log2, bh = 1 << g.bh_log2;
  const int b = (y >> g.bh_log2) * g.binsX + (x >> g.bw_log2);
  const int r = b % g.nranks, k = b / g.nranks;
  const int p = (y & (bh - 1)) * bw + (x & (bw - 1));
  const unsigned long long key =
      a.all_keys[((size_t)r * a.owned_max + k) * (size_t)(bw * bh) + p];
  float L[3];
  normalise_light(a.light, L);
  const size_t o = (size_t)y * g.W + x;
  float4 c = make_float4(0.f, 0.f, 0.f, 0.f);
  float depth = 1.0f;
  int prim = -1;
  if (key != CLEAR_KEY) {
    prim = (int)(unsigned)(key & 0xFFFFFFFFu);
    depth = __uint_as_float((unsigned)(key >> 32));
    c = shade(a.verts, a.idx, a.M, g.W, g.H, L, prim, 256 * x + 128, 256 * y + 128);
  }
  reinterpret_cast<float4*>(a.out_rgba)[o] = c;
  a.out_depth[o] = depth;
  a.out_primid[o] = prim;
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
cudaError_t launch_setup(const SetupArgs& a, int grid, cudaStream_t s) {
  k_setup<<<grid, K1_THREADS, 0, s>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_bin_scan(const ScanArgs& a, int grid, cudaStream_t s) {
  k_bin_scan<<<grid, SCAN_THREADS, 0, s>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_radix_pass(const RadixArgs& a, int grid, cudaStream_t s) {
  k_radix_pass<<<grid, RX_THREADS, 0, s>>>(a);
  return cudaGetLastError();
}

template <int BW, int BH>
static cudaError_t launch_tile_t(const TileArgs& a, int nb, bool cov, bool keys_only, cudaStream_t s) {
  constexpr int NPX = BW * BH;
  constexpr int THREADS = NPX < 256 ? NPX : 256;
  size_t smem = (size_t)NPX * 8 + (size_t)THREADS * (48 + 4) + (cov ? (size_t)NPX * 4 : 0);
  auto run = [&](auto kern) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<nb, THREADS, smem, s>>>(a);
    return cudaGetLastError();
  };
  if (keys_only) return cov ? run(k_tile<BW, BH, THREADS, true, true>) : run(k_tile<BW, BH, THREADS, false, true>);
  return cov ? run(k_tile<BW, BH, THREADS, true, false>) : run(k_tile<BW, BH, THREADS, false, false>);
}

#define PIKO_TILE_CASE(W_, H_) \
  if (bw == W_ && bh == H_) return launch_tile_t<W_, H_>(a, nb, cov, keys_only, s);

cudaError_t launch_tile(const TileArgs& a, int bw, int bh, int nb, bool cov, bool keys_only,
                        cudaStream_t s) {
  if (nb <= 0) return cudaSuccess;
  PIKO_TILE_CASE(8, 8) PIKO_TILE_CASE(8, 16) PIKO_TILE_CASE(8, 32) PIKO_TILE_CASE(8, 64)
  PIKO_TILE_CASE(16, 8) PIKO_TILE_CASE(16, 16) PIKO_TILE_CASE(16, 32) PIKO_TILE_CASE(16, 64)
  PIKO_TILE_CASE(32, 8) PIKO_TILE_CASE(32, 16) PIKO_TILE_CASE(32, 32) PIKO_TILE_CASE(32, 64)
  PIKO_TILE_CASE(64, 8) PIKO_TILE_CASE(64, 16) PIKO_TILE_CASE(64, 32) PIKO_TILE_CASE(64, 64)
  return cudaErrorInvalidValue;
}

cudaError_t launch_resolve(const ResolveArgs& a, cudaStream_t s) {
  dim3 grid((a.g.W + 31) / 32, (a.g.H + 7) / 8);
  k_resolve<<<grid, 256, 0, s>>>(a);
  return cudaGetLastError();
}

static int occ_grid(const void* f, int threads, size_t smem) {
  int dev = 0, sms = 148, occ = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, f, threads, smem);
  return sms * (occ > 0 ? occ : 1);
}
int max_grid_setup() { return occ_grid((const void*)k_setup, K1_THREADS, 0); }
int max_grid_scan() { return occ_grid((const void*)k_bin_scan, SCAN_THREADS, 0); }
int max_grid_radix() { return occ_grid((const void*)k_radix_pass, RX_THREADS, 0); }

}  // namespace piko
