// piko_internal.h -- structures shared by the kernels (kernels.cu) and the host
// orchestration (piko_api.cu).  Product code only; nothing here is shared with
// the CPU checker.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace piko {

// ---- launch geometry -------------------------------------------------------
constexpr int K1_THREADS = 256;                     // triangle-setup CTA
#ifndef PIKO_K1_TPT
#define PIKO_K1_TPT 4
#endif
constexpr int K1_TPT = PIKO_K1_TPT;                 // triangles per thread (strided)
constexpr int K1_CHUNK = K1_THREADS * K1_TPT;       // triangles per CTA
// the host sizes count-matrix rows from 2^10 = K1_CHUNK triangles and the
// chunk-list groups from 32 per warp slot; other chunk sizes are not supported
// (K1_TPT = 1 / 2 builds fail at run time)
static_assert(K1_CHUNK == 1024, "k_setup handles 1024 triangles per CTA");
constexpr int EX_MAX_TRIS = 4096;                   // triangles per expand chunk (radix pass 0)
#ifndef PIKO_RX_THREADS
#define PIKO_RX_THREADS 256
#endif
constexpr int SCAN_THREADS = PIKO_RX_THREADS;       // bin-count scan (run by radix-pass CTAs: == RX_THREADS)
constexpr int SCAN_ITEMS = 4;
constexpr int SCAN_CHUNK = SCAN_THREADS * SCAN_ITEMS;
constexpr int RX_THREADS = PIKO_RX_THREADS;         // stable LSD radix pass CTA
constexpr int RX_MIN_CTAS = 2;                      // resident per SM (shared memory allows 2)
constexpr int RX_WARPS = RX_THREADS / 32;
constexpr int RX_ITEMS = 4096 / RX_THREADS;        // RX_CHUNK = 4096 pairs
constexpr int RX_CHUNK = RX_THREADS * RX_ITEMS;     // pairs per chunk
constexpr int RX_BITS = 8;
static_assert(SCAN_THREADS == RX_THREADS && RX_THREADS >= (1 << RX_BITS), "digit-owner threads");
constexpr int LB_GROUP = 16;                        // chunks per look-back group
constexpr int RX_RADIX = 1 << RX_BITS;
constexpr int MAX_PASSES = 3;                       // NB <= 2^24 bins
constexpr unsigned long long MAX_PAIRS = 1ull << 31;  // bin_start is int32
// Schedule: the bin scan builds k_tile's work lists.  A bin with more than
// `frag` pairs is split into fragments of `frag` consecutive CSR entries that
// different CTAs rasterize and merge into a global key tile (64-bit atomicMin);
// the last fragment to arrive shades the bin.  Lists: [0] fragments of split
// bins, [1 .. SIZE_CLASSES] single-fragment bins by size class (pairs >
// 3/4, 1/2, 1/4 of a fragment, rest), [NLIST-1] empty bins.  k_tile drains
// them in that order: largest work first (an LPT approximation without a sort,
// so a CTA left with a second item gets a small one).
constexpr int SIZE_CLASSES = 4;
constexpr int NLIST = 2 + SIZE_CLASSES;
constexpr int LIST_EMPTY = NLIST - 1;
#ifndef PIKO_FRAG_ROUNDS
#define PIKO_FRAG_ROUNDS 4
#endif
constexpr int FRAG_ROUNDS = PIKO_FRAG_ROUNDS;  // fragment = FRAG_ROUNDS * threads-per-CTA pairs
constexpr int EMPTY_GROUP = 8;   // empty bins per k_tile queue ticket
constexpr int OVQ_CAP = 1024;
// Count-matrix AssignBin: used when NB <= CM_MAX_NB and the
// matrix of rows x NB per-row bin counts stays below CM_MAX_ENTRIES.
constexpr int CM_MAX_NB = 32768;                 // touched-bin bitmap in shared memory
constexpr long long CM_MAX_ENTRIES = 1ll << 24;  // rows * NB
constexpr int CM_SUB = 4096;                     // triangles per scatter sub-chunk (registers)
constexpr int CM_COLS = 16;                      // k_cm_scan: bins per CTA (x 16 row groups)
// Chunk-list AssignBin (round 2): each k_setup CTA (a chunk
// of K1_CHUNK triangles = 32 groups of 32) records per touched bin the mask of
// its groups with a pair in the bin and the pair count; k_cl_bins walks a bin's
// chunks (bitmap) and groups (masks) in primitive order and compacts the
// triangles whose rect holds the bin with warp ballots.
constexpr int CL_MAX_NB = 4096;                  // per-bin masks / counts of a chunk in shared memory
constexpr int CL_WPT = 8;                        // bitmap words per k_cl_bins thread (chunks <= 512*32*8)
constexpr long long CL_MAX_ENTRIES = 1ll << 26;  // NB x chunks (the entry matrix)
constexpr int CLB_THREADS = 256;                 // k_cl_bins CTA
constexpr int CLB_ENT = 1024;                    // entries (chunks) of one bin (more: count matrix)
constexpr int CLB_GRP = 2048;                    // groups of one bin (more: count matrix)
constexpr int CLB_KMAX = 32;                     // bins per persistent k_cl_bins CTA

// ---- persistent device control block ----------------------------------------
// Never memset per frame: every kernel of a frame takes exactly gridDim.x
// tickets from its counter, so  frame = ticket / gridDim.x  and
// chunk = ticket % gridDim.x.  Look-back status words carry the tag frame+1.
// Per-frame accumulators are double-buffered by frame parity; the tile kernel
// zeroes the next frame's copy.  The host resets the block (and the status
// arrays) only when a grid size changes or after an error.
struct Control {  // (the mirror copies whole 8-byte words up to digit_hist: keep u32 fields paired)
  unsigned long long k1_ticket;
  unsigned long long rx_ticket[MAX_PASSES];
  unsigned long long scan_ticket;      // standalone bin-scan kernel (single-pass grids)
  unsigned long long cm_done;          // k_cm_scan CTAs finished (modulo grid: the last scans bin_start)
  unsigned long long cl_done;          // chunk-list k_setup CTAs finished (modulo grid: the last scans bin_start)
  unsigned long long cm_touched;       // count-matrix frame: sum over scatter windows of the bins touched
                                       //   (dense rows, e.g. unordered soups: the host switches to the radix passes)
  unsigned long long frame;            // written by K1 chunk 0
  unsigned int tile_next;              // dynamic bin queue of k_tile (reset by K1 chunk 0)
  unsigned int list_n[NLIST];          // work-list sizes (reset by K1 chunk 0)
  unsigned int empty_next;             // k_tile queue of empty-bin groups (reset by K1 chunk 0)
  unsigned int eq_next;                // k_tile ticket queue over all bins for the empty ones (reset by K1 chunk 0)
  unsigned int vmax;                   // max(idx)+1 from k_index_max (zeroed by K1 chunk 0)
  unsigned int vx_overflow;            // k_vertex: vmax > xv capacity (K1 turns it into overflow_tag)
  unsigned long long vx_need;          // vertex count the last frame needed
  unsigned long long n_pairs;          // P, written by K1's last chunk
  unsigned long long overflow_tag;     // frame+1 of the last frame whose P > capacity
  unsigned long long n_live[2];        // parity double buffer (statistics)
  unsigned long long p2p_arrive;       // k_tile CTA tickets (P2P arrival, modulo grid)
  unsigned long long p2p_count;        // k_resolve CTA tickets (P2P slot release)
  unsigned int p2p_timeout;            // a peer flag wait timed out (sticky)
  unsigned int cl_overflow;            // a bin had more than CLB_ENT chunks / CLB_GRP groups (host: count matrix)
  unsigned long long peer_overflow;    // rank 0: frame+1 of a frame in which a peer rank overflowed
  unsigned long long tile_done;        // (unused since k_tile CTA 0 writes the host mirror at its start)
  unsigned int digit_hist[2][MAX_PASSES][RX_RADIX];  // parity double buffer
};

static_assert(offsetof(Control, digit_hist) % 8 == 0, "the host mirror copies whole words");

struct Mat4 {
  float m[16];
};

// Screen / bin grid / ownership, identical for every kernel of a frame.
struct Grid {
  int W, H;
  int bw_log2, bh_log2;
  int binsX, binsY, NB;
  int rank, nranks;     // sort-first ownership: bin b belongs to b % nranks
};

// Setup record of one live triangle: 48 bytes = 3 x int4.
//   q0 = {X0, Y0, X1, Y1}                 snapped corners (subpixels, 16.8)
//   q1 = {X2, Y2, bits(zw0), bits(za)}    z plane z = zw0 + za*dX + zb*dY
//   q2 = {bits(zb), px0|py0<<16, px1|py1<<16, flags}  sample-centre pixel rect
// flags bit 0: bbox extent < 2^15 subpixels in x and y -> int32 edge path.
constexpr int REC_SMALL = 1;

// Vertex stage output, one per vertex (16 B): snapped X, Y (subpixels),
// bits(zw), bits(rw); X == VX_CULLED marks a corner that culls its triangles.
constexpr int VX_CULLED = (int)0x80000000;
constexpr int VX_THREADS = 256;
#ifndef PIKO_VX_VPT
#define PIKO_VX_VPT 4
#endif
constexpr int VX_VPT = PIKO_VX_VPT;             // vertices per k_vertex thread (loads issued together)

struct VertexArgs {
  const float* verts;
  long long n_verts;            // < 0: read ctl->vmax (piko_draw without a count)
  long long cap;                // xv capacity
  Control* ctl;
  Mat4 M;
  int W, H;
  int4* xv;                     // [n_verts] transformed vertices
};

struct SetupArgs {
  const int4* xv;               // transformed vertices; null: fused vertex stage (below)
  long long xv_cap;             // corners with idx >= xv_cap are culled (overflowed frame)
  const float* verts;           // fused mode: corners transformed here from verts ...
  Mat4 M;                       // ... with M (same O1 arithmetic as k_vertex)
  const int32_t* idx;
  long long n_tris;
  Grid g;
  int npass;                    // radix digit histograms to build (0 in count-matrix mode)
  uint32_t* cm;                 // count-matrix AssignBin: M[n_tris >> cm_shift][NB] (null: radix mode)
  int cm_shift;                 // log2 triangles per count-matrix row
  unsigned long long frame;     // frames enqueued since the control block was reset (host counter)
  int4* rec;                    // 3 x 16 B per triangle (rec_at: [3][rec_stride] or [n_tris][3])
  long long rec_stride;         // triangles per record plane (the record capacity)
  uint2* rect;                  // [n_tris] tile rect {tx0|ty0<<16, tx1|ty1<<16}; empty if culled
  Control* ctl;
  // chunk-list AssignBin (null: off): per touched bin b, cl_ent[b][chunk] =
  // {mask of the chunk's 32-triangle groups with a pair in b, pairs}, bit
  // `chunk` of cl_bm[b][cl_nw], cl_tot[b] += pairs
  uint2* cl_ent;
  uint32_t* cl_bm;
  uint32_t* cl_tot;             // this frame's parity half of [2][NB]
  long long cl_nch;             // chunks (= grid)
  int cl_nw;                    // bitmap words per bin
  int32_t* cl_start;            // [NB+1] bin_start: the grid's last CTA scans the totals
  unsigned long long cl_cap;    //   ... and checks P against the pair capacity
};

struct RadixArgs {
  // pass 0 expands the (bin, primID) pairs of a chunk of triangles from rects
  int expand;
  const uint2* rect;
  long long n_tris;
  int tri_chunk;                // triangles per expand chunk (<= EX_MAX_TRIS)
  Grid g;
  unsigned long long cap;       // pair capacity (pass 0 checks P against it)
  int scan_here;                // extra CTAs of this launch run the bin scan
  const uint32_t* keys_in;
  const int32_t* vals_in;
  uint32_t* keys_out;           // may be null on the last pass
  int32_t* vals_out;
  unsigned long long* status;   // [sort chunks][RX_RADIX] chunk look-back words
  unsigned long long* gstatus;  // [groups][RX_RADIX] group look-back words
  uint32_t* ccount;             // [sort chunks][RX_RADIX] per-chunk digit counts
  uint32_t* garrive;            // [2][gcap] chunks of a group that published (by frame parity)
  long long gcap;               // group capacity
  Control* ctl;
  int pass;
  int shift;
  // bin scan (pass 0 only): extra CTAs after the sort chunks
  uint32_t* bin_count;
  int32_t* bin_start;
  unsigned long long* scan_status;  // [scan tiles]
  int NB;
  int rank, nranks;             // only owned bins enter the work lists
  int2* frag_list;              // [frag_cap] {bin, fragment}
  int32_t* bin_list;            // [NLIST-1][NB] single-fragment bins by size class, empty bins
  uint32_t* gcov;               // [NB][bw*bh] coverage tiles (debug) or null
  int frag;                     // pairs per fragment
  int npx;                      // pixels per bin
};

// Count-matrix AssignBin (a3-a6 for NB <= CM_MAX_NB): k_setup adds each
// triangle's owned bins into row t >> cm_shift of M; k_cm_scan turns M into
// per-row exclusive column prefixes CP[r][b] = bin_start[b] + sum_{r' < r}
// M[r'][b] and the bin totals, its last CTA bin_start and P; k_cm_scatter
// writes every row's pairs at bin_start[b] + CP[r][b] + (stable rank inside
// the row).  The bin scan work lists reuse
// RadixArgs (extra CTAs of k_cm_scatter).
struct CmArgs {
  uint32_t* cm;                 // [rows][NB] counts (zeroed again by k_cm_scan)
  uint32_t* cp;                 // [rows][NB] column prefixes / running cursors
  long long rows;
  int cm_shift;
  const uint2* rect;
  long long n_tris;
  Grid g;
  unsigned long long cap;       // pair capacity
  int32_t* bin_prims;           // [P] output CSR values
  Control* ctl;
  RadixArgs sched;              // bin_start, work lists (schedule CTAs)
};

// Chunk-list AssignBin, second half (k_cl_bins): persistent CTAs take the
// non-empty bins; a bin's chunk bitmap (ascending chunk) and group masks
// (ascending group) enumerate its candidate triangles in primitive order, the
// rect test + ballot compacts them to bin_prims[bin_start[b] ...].  Extra CTAs
// build k_tile's work lists.
struct ClArgs {
  const uint2* cl_ent;
  const uint2* rect;
  uint32_t* cl_bm;              // words are zeroed after reading (next frame)
  uint32_t* cl_tot;             // [2][NB]: this frame's parity read, the other zeroed
  long long nch;
  int nw;
  int nbin_ctas;                // CTAs of the gather part (the rest build work lists)
  long long n_tris;
  unsigned long long frame;     // host frame counter (parity of cl_tot)
  Grid g;
  unsigned long long cap;       // pair capacity of bin_prims
  int32_t* bin_prims;
  Control* ctl;
  RadixArgs sched;              // bin_start, work lists (schedule CTAs)
};

// Pixel-shader complexity: `iters` extra
// dependent FMAs per shaded fragment -- forward: every covered fragment that
// passes the depth range pays them inside the raster loop (the paper's
// pipelines shade before the depth test); deferred: once per resolved
// pixel.  The result only reaches `sink` on an impossible branch (it is
// always >= 0), so images are bit-identical for every setting.
struct ShaderCost {
  int iters;                    // 0: off
  int forward;                  // 1: per fragment, 0: per pixel
  float* sink;                  // never written in practice (result < 0 only)
};

struct TileArgs {
  const float* verts;
  const int4* xv;               // null: shade re-transforms corners from verts with M
  Mat4 M;
  const int32_t* idx;
  float light[3];
  Grid g;
  int npass;
  const int4* rec;
  long long rec_stride;
  int32_t* bin_start;           // written here only when npass == 0 (NB == 1)
  const int32_t* bin_prims;
  Control* ctl;
  float* out_rgba;              // may be null (keys-only mode)
  float* out_depth;
  int32_t* out_primid;
  uint32_t* out_cov;            // debug coverage counts or null
  unsigned long long* tile_keys;  // keys-only mode: [owned][bw*bh]
  int owned;                    // bins owned by this rank (grid may be larger)
  const int2* frag_list;
  const int32_t* bin_list;
  unsigned long long* fkey;      // [frag_cap][bw*bh] key tile of every fragment item (slot = item index)
  uint32_t* gcov;
  uint32_t* arrive;             // [NB] fragments merged so far (self-resetting)
  int frag;
  uint32_t* garrive;            // [npass][2][gcap] look-back group arrival counters;
  long long gcap;               //   k_tile zeroes the next frame's parity
  unsigned prim_base;           // keys-only: added to the primID of every stored key (sort-last)
  int radix;                    // 1: the frame used the radix AssignBin (its look-back counters)
  int skip_empty;               // 1: bins without pairs are not written (the deferred resolve knows them)
  int early_empty;              // 1: empty bins (bin_count == 0) from one ticket queue, drained first by
                                //    the CTAs resident before the dependency wait (count-matrix frames)
  const uint32_t* bin_count;    // [NB] pair counts (early_empty)
  Control* status_out;          // mapped host mirror: the last CTA copies the control block (null: none)
  int4* ovq;                    // [grid][OVQ_CAP][6] overflow of the per-bin queue (null: none)
  // P2P transport (sort-first): tile_keys points into rank 0's memory
  unsigned long long* p2p_flag;         // rank 0's arrival flag of this rank (null: no P2P)
  const unsigned long long* p2p_done;   // rank 0's last resolved epoch
  unsigned long long epoch;             // this frame's exchange epoch (1, 2, ...)
  ShaderCost sc;
  unsigned long long* status_word;      // multi-GPU: this rank's frame status next to its keys (null: none)
  unsigned long long status_ok;         //   value meaning "no overflow" (NCCL: 1; P2P: the epoch)
};

struct ResolveArgs {            // rank 0 after the NCCL gather
  const float* verts;
  const int4* xv;
  Mat4 M;
  const int32_t* idx;
  float light[3];
  Grid g;
  const unsigned long long* all_keys;  // [nranks][owned_max][bw*bh]
  int owned_max;
  float* out_rgba;
  float* out_depth;
  int32_t* out_primid;
  // P2P transport: wait for every rank's arrival flag, then release the slot
  const unsigned long long* p2p_flags;  // [nranks] (null: keys already local)
  unsigned long long* p2p_done;
  unsigned long long* p2p_count;        // CTA ticket (self-resetting modulo grid)
  unsigned* p2p_timeout;
  unsigned long long epoch;
  ShaderCost sc;                         // deferred shader cost (single-GPU deferred resolve)
  long long rank_stride;                 // words between ranks' key blocks (0: owned_max*bw*bh)
  const unsigned long long* status;      // ranks' status words (null: none), status_stride apart
  long long status_stride;
  int nstatus;
  unsigned long long status_ok;
  Control* ctl;                          // rank 0: peer_overflow is raised here
  const int32_t* bin_start;              // single-GPU deferred resolve: [NB+1] (empty bins: background) or null
};

// FreePipe variant (sec. 7.2.1): one fused
// kernel, one thread per triangle, global 64-bit atomicMin into a full-screen
// key buffer, then a per-pixel resolve/shade pass.
struct FreePipeArgs {
  const float* verts;
  const int4* xv;               // null: fused vertex stage (corners transformed in k_freepipe)
  Mat4 M;
  long long xv_cap;
  const int32_t* idx;
  long long n_tris;
  int W, H;
  unsigned long long* keys;     // [H][W], CLEAR between frames (resolve resets)
  uint32_t* cov;                // debug coverage counts or null
  float light[3];
  float* out_rgba;
  float* out_depth;
  int32_t* out_primid;
  ShaderCost sc;
};

// Baseline design alternative (sec. 7.1,
// P:404-410): one kernel per stage of VS -> Rasterizer -> Fragment Shader ->
// Depth Test -> Composite with full-screen bins and LoadBalance (thread per
// primitive / per fragment), every stage reading and writing off-chip memory.
struct BaselineArgs {
  const float* verts;
  const int4* xv;               // vertex-stage records (the VS kernel always runs)
  long long xv_cap;
  Mat4 M;
  const int32_t* idx;
  long long n_tris;
  int W, H;
  float light[3];
  unsigned long long* keys;      // [H][W] depth buffer, CLEAR between frames
  unsigned long long* frag_key;  // [frag_cap] fragment (depth, primID) keys
  uint32_t* frag_px;             // [frag_cap] fragment pixel index y*W + x
  float4* frag_rgba;             // [frag_cap] shaded fragment colours
  long long frag_cap;
  unsigned long long* n_frag;    // fragments emitted this frame (may exceed frag_cap)
  uint32_t* cov;                 // debug coverage counts or null
  float* out_rgba;
  float* out_depth;
  int32_t* out_primid;
  ShaderCost sc;
};

// Reyes Split + Dice (R19-R21): bicubic Bezier
// patches -> micropolygon mesh that the binned pipeline then samples (32x32
// bins).
struct DiceArgs {
  const float* patches;          // f32[n][16][4] (x, y, z, pad), control point a*4+b
  long long n;
  Mat4 M;
  int W, H;
  float dice_px;
  int max_grid;
  int2* rate;                    // [n] (Gu, Gv)
  long long* base;               // [n][2] first vertex, first triangle
  long long* total;              // [2] vertices, triangles (device; copied to the host)
  float* verts;                  // [V][8] out
  int32_t* idx;                  // [T][3] out
};

// ---- launchers (kernels.cu); pdl = programmatic dependent launch -----------
cudaError_t launch_dice_rate(const DiceArgs& a, cudaStream_t s);
cudaError_t launch_dice(const DiceArgs& a, cudaStream_t s);
cudaError_t launch_baseline(const BaselineArgs& a, int stage, bool pdl, cudaStream_t s);
cudaError_t launch_freepipe(const FreePipeArgs& a, bool pdl, cudaStream_t s);
cudaError_t launch_fp_resolve(const FreePipeArgs& a, bool pdl, cudaStream_t s);
cudaError_t launch_index_max(const int32_t* idx, long long n, Control* ctl, bool pdl, cudaStream_t s);
cudaError_t launch_vertex(const VertexArgs& a, bool pdl, cudaStream_t s);
cudaError_t launch_setup(const SetupArgs& a, int grid, bool pdl, cudaStream_t s);
cudaError_t launch_radix_pass(const RadixArgs& a, int grid, bool pdl, cudaStream_t s);
cudaError_t launch_bin_scan(const RadixArgs& a, int grid, bool pdl, cudaStream_t s);
cudaError_t launch_cm_scan(const CmArgs& a, int grid, bool pdl, cudaStream_t s);
cudaError_t launch_cm_scatter(const CmArgs& a, int grid, bool pdl, cudaStream_t s);
cudaError_t launch_cl_bins(const ClArgs& a, int grid, bool pdl, cudaStream_t s);
inline int cm_scan_grid(int NB) { return (NB + CM_COLS - 1) / CM_COLS; }
cudaError_t launch_tile(const TileArgs& a, int bw, int bh, int grid, bool cov, bool keys_only,
                        bool pdl, cudaStream_t s);
int tile_grid(int bw, int bh, bool cov, bool keys_only);  // persistent grid size
struct TileKernel {
  void (*fn)(TileArgs) = nullptr;
  int threads = 0;
  size_t smem = 0;
};
TileKernel tile_kernel_bw8(int bh, bool cov, bool keys_only);   // k_tile instantiation of a bin shape
TileKernel tile_kernel_bw16(int bh, bool cov, bool keys_only);
TileKernel tile_kernel_bw32(int bh, bool cov, bool keys_only);
TileKernel tile_kernel_bw64(int bh, bool cov, bool keys_only);
#ifndef PIKO_TILE_THREADS
#define PIKO_TILE_THREADS 256
#endif
constexpr int TILE_THREADS = PIKO_TILE_THREADS;  // k_tile CTA size cap
inline int tile_threads(int bw, int bh) { return bw * bh < TILE_THREADS ? bw * bh : TILE_THREADS; }
inline int tile_frag(int bw, int bh) { return FRAG_ROUNDS * tile_threads(bw, bh); }
cudaError_t launch_resolve(const ResolveArgs& a, bool pdl, cudaStream_t s);
cudaError_t launch_shade(const ResolveArgs& a, bool pdl, cudaStream_t s);  // single-GPU deferred resolve

}  // namespace piko
