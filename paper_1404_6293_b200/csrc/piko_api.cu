// piko_api.cu -- host orchestration behind the C ABI of include/piko.h.
//
// One piko_ctx = one framebuffer shape + bin grid on one device.  It owns the
// per-frame scratch (setup records, pair lists, bin CSR, look-back status
// words, primID / coverage buffers), grows it on demand, enqueues the kernel
// sequence of a frame on the caller's stream, and (multi-GPU) runs the NCCL
// tile-key gather to rank 0.  See DESIGN.md "Boundary" and "Host runtime".
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/piko.h"
#include "piko_internal.h"

using namespace piko;

// ---------------------------------------------------------------------------
// minimal run-time NCCL binding (dlopen libnccl.so.2; reuses torch's copy if
// it is already loaded).  Only the calls of the tile gather are bound.
// ---------------------------------------------------------------------------
namespace {
typedef struct ncclComm* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef int ncclResult_t;
enum { ncclUint8_ = 1, ncclUint64_ = 5 };  // ncclDataType_t values
enum { ncclMin_ = 3 };                      // ncclRedOp_t value

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Reduce)(const void*, void*, size_t, int, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  bool load(std::string& err) {
    if (h) return true;
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) { err = "cannot dlopen libnccl.so.2"; return false; }
#define PIKO_SYM(n) n = reinterpret_cast<decltype(n)>(dlsym(h, "nccl" #n)); if (!n) { err = "missing nccl" #n; return false; }
    PIKO_SYM(CommInitRank) PIKO_SYM(CommDestroy) PIKO_SYM(Send) PIKO_SYM(Recv) PIKO_SYM(Reduce) PIKO_SYM(Broadcast)
    PIKO_SYM(GroupStart) PIKO_SYM(GroupEnd) PIKO_SYM(GetErrorString) PIKO_SYM(GetUniqueId)
#undef PIKO_SYM
    return true;
  }
};
Nccl g_nccl;

thread_local std::string g_create_error;

int ilog2(int v) { int l = 0; while ((1 << l) < v) ++l; return l; }
bool pow2_in(int v, int lo, int hi) { return v >= lo && v <= hi && (v & (v - 1)) == 0; }
}  // namespace

struct piko_ctx {
  int device = 0;
  int sms = 148;            // multiprocessors of this context's device
  Grid g{};
  int bw = 0, bh = 0;
  int npass = 0;
  int owned = 0;            // bins owned by this rank
  unsigned debug = 0;
  int sync_mode = PIKO_SYNC_ASYNC;   // piko_draw returns once enqueued
  bool virt = false;        // virtual rank (partition without communicator)
  int multi = PIKO_MULTI_SORT_FIRST;
  int mrank = 0, mnranks = 1;  // multi-GPU rank / size (sort-last: g.rank = 0, g.nranks = 1)
  long long prim_base = 0;     // sort-last: first triangle of this rank's range
  // P2P transport (sort-first): rank 0 owns the exchange buffers; the other
  // ranks map them (CUDA IPC over NVLink, or the same pointers for virtual
  // ranks on one device) and k_tile stores its keys straight into them
  int transport = PIKO_XPORT_NCCL;
  unsigned long long* p2p_keys = nullptr;  // rank 0: [2][nranks][owned_max][bw*bh]
  unsigned long long* p2p_sync = nullptr;  // rank 0: [nranks] arrival epochs + [1] done epoch
  bool p2p_owner = false, p2p_ipc = false;
  unsigned long long epoch = 0;            // exchange epoch of the last frame
  std::string err;

  // scratch
  int4* rec = nullptr; long long rec_cap = 0;
  int4* xv = nullptr; long long xv_cap = 0;   // vertex-stage records
  uint32_t* keys[2] = {nullptr, nullptr};
  int32_t* vals[2] = {nullptr, nullptr};
  unsigned long long pair_cap = 0;
  uint32_t* bin_count = nullptr;
  int32_t* bin_start = nullptr;
  int2* frag_list = nullptr; long long frag_cap = 0;  // split-bin fragments
  int32_t* bin_list = nullptr;       // [NLIST-1][NB] single-fragment bins by size class, empty bins
  unsigned long long* fkey = nullptr;  // [frag_cap][bw*bh] key tile of every split-bin fragment
  uint32_t* gcov = nullptr;          // [NB][bw*bh] coverage tiles (debug)
  uint32_t* arrive = nullptr;        // [NB] fragment arrival counters
  int4* ovq = nullptr; long long ovq_ctas = 0;  // k_tile queue overflow [ctas][OVQ_CAP][6]
  Control* ctl = nullptr;
  uint2* rect = nullptr;                 // [rec_cap] tile rect per triangle
  int tri_chunk = EX_MAX_TRIS;           // triangles per expand chunk (adapted to P/T)
  unsigned long long* st_scan = nullptr; long long st_scan_n = 0;
  unsigned long long* st_rx = nullptr; long long st_rx_chunks = 0;  // [npass][chunks][256]
  unsigned long long* st_grp = nullptr;   // [npass][groups][256] group look-back words
  uint32_t* ccount = nullptr;             // [npass][chunks][256] per-chunk digit counts
  uint32_t* garr = nullptr;               // [npass][2][groups] group arrival counters
  long long gcap = 0;
  // grid sizes of the last frame: the ticket/tag scheme of Control needs them
  // constant, so a change forces a reset of the control block + status words
  long long last_grids[6] = {-1, -1, -1, -1, -1, -1};
  bool need_reset = true;
  unsigned long long frames = 0;      // binned frames enqueued since the control block was reset
  bool pdl = true;
  int vs_mode = -1;        // vertex stage: -1 auto, 0 fused into k_setup, 1 separate k_vertex
  int32_t* primid = nullptr;
  uint32_t* cov = nullptr;
  // Asynchronous frames (piko_draw returns once enqueued).  Each
  // enqueued frame copies its control block into a pinned mirror of a ring
  // slot and records an event; a frame's status is evaluated when its event
  // has completed -- polled without blocking at the next draw, waited for
  // only when the ring is full, at piko_finish, or by an inspection call.
  static constexpr int NRING = 8;
  struct Slot {
    Control* h = nullptr;   // pinned, mapped host mirror
    Control* d = nullptr;   // its device alias: the binned frame's last kernel writes it directly
    cudaEvent_t ev = nullptr;
    long long T = 0;
    bool cm = false;        // the frame used the count-matrix AssignBin
  };
  Slot ring[NRING];
  int ring_head = 0, ring_n = 0;     // next slot to fill; frames in flight
  Control* h_ctl = nullptr;          // mirror of the last evaluated frame
  bool pending = false;              // ring_n > 0
  int last_status = PIKO_OK;         // status of the last evaluated frame
  int sticky = PIKO_OK;              // first error of an async frame not yet returned
  long long last_T = 0;
  int last_kernels = 0;                // kernels launched by the last frame


  // Reyes Split/Dice output (piko_draw_patches): the micropolygon mesh
  float* dice_verts = nullptr; long long dice_vcap = 0;
  int32_t* dice_idx = nullptr; long long dice_tcap = 0;
  int2* dice_rate = nullptr; long long* dice_base = nullptr; long long dice_pcap = 0;
  long long* dice_total = nullptr;        // device [2]
  long long* h_dice_total = nullptr;      // pinned [2]
  long long dice_V = 0, dice_T = 0;

  // pipelined end-to-end staging (piko_draw_host_async): two slots, an upload
  // and a download stream; a slot is reused once its previous frame is drawn
  struct HostSlot {
    float* verts = nullptr; long long vcap = 0;
    int32_t* idx = nullptr; long long icap = 0;
    float* rgba = nullptr; float* depth = nullptr;
    cudaEvent_t in_done = nullptr, frame_done = nullptr, out_done = nullptr;
    bool used = false;
  };
  HostSlot hs[2];
  int hs_next = 0;
  cudaStream_t cs_in = nullptr, cs_out = nullptr;
  // end-to-end staging
  float* d_verts = nullptr; long long d_verts_cap = 0;
  int32_t* d_idx = nullptr; long long d_idx_cap = 0;
  float* d_rgba = nullptr; float* d_depth = nullptr;

  // multi-GPU
  ncclComm_t comm = nullptr;
  unsigned long long* tile_keys = nullptr;  // [owned_max][bw*bh]
  unsigned long long* all_keys = nullptr;   // rank 0: [nranks][owned_max][bw*bh]
  int owned_max = 0;
  bool keys_mode = false;                   // inside piko_draw_tile_keys
  // single GPU: k_tile writes packed keys only and a separate full-occupancy
  // k_resolve shades the frame (removes the per-pixel dependent shading
  // gathers from the per-bin critical path of k_tile)
  int deferred = 0;
  // count-matrix AssignBin (NB <= CM_MAX_NB; radix passes otherwise)
  int cm_mode = -1;                         // -1 auto, 0 radix, 1 count matrix
  int cm_tc_log2 = 0;                       // forced log2 triangles per row (0: auto)
  uint32_t* cm = nullptr; uint32_t* cp = nullptr; long long cm_cap = 0;  // [rows][NB]
  bool tile_items_grid = false;             // k_tile: one CTA per possible item instead of persistent
  bool last_cm = false;                     // the last frame used the count matrix
  long long cm_dense_T = -1;                 // triangle count of frames whose count matrix was dense
  long long last_cm_rows = 0;
  // chunk-list AssignBin (NB <= CL_MAX_NB; the default where it applies)
  int early_empty = 1;                      // PIKO_EARLY_EMPTY=0: empty bins after the pair items
  int cl_mode = 0;                          // 0 off (default: slower on c2/c3), 1 on where it applies
  bool cl_off = false;                      // a chunk overflowed CL_WIN: count matrix from now on
  bool last_cl = false;                     // the last frame used the chunk lists
  long long last_cl_nch = 0;
  uint2* cl_ent = nullptr; long long cl_ent_cap = 0;      // [NB][chunks] {group mask, pairs}
  uint32_t* cl_bm = nullptr; long long cl_bm_cap = 0;     // [NB][words]
  uint32_t* cl_tot = nullptr;                              // [2][NB]
  int32_t* prims_out = nullptr;             // CSR bin_prims of the last frame
  unsigned long long* def_keys = nullptr;   // [NB][bw*bh]
  int pipeline = PIKO_PIPE_BINNED;
  unsigned long long* fp_keys = nullptr;    // FreePipe full-screen key buffer
  ShaderCost sc{};                          // pixel-shader complexity knob (NEXT-3)
  // Baseline pipeline (NEXT-3): full-screen depth buffer + fragment buffers
  unsigned long long* bl_keys = nullptr;    // [H][W]
  unsigned long long* frag_key = nullptr;   // [bl_cap]
  uint32_t* frag_px = nullptr;
  float4* frag_rgba = nullptr;
  long long bl_cap = 0;                     // Baseline fragment capacity

  // profiling: PIKO_NUM_STAGES + 1 boundary events per frame
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  long long prof_frames = 0;
  cudaEvent_t* frame_events() {
    const size_t need = (size_t)(prof_frames + 1) * (PIKO_NUM_STAGES + 1);
    while (ev_pool.size() < need) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
      ev_pool.push_back(e);
    }
    return &ev_pool[(size_t)prof_frames * (PIKO_NUM_STAGES + 1)];
  }

  int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    err = buf;
    return code;
  }
};

#define CK(call)                                                                    \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess)                                                          \
      return ctx->fail(PIKO_ECUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                       __FILE__, __LINE__);                                         \
  } while (0)

extern "C" int64_t piko_owned_bins(int, int, int, int, int, int, int32_t*, int64_t);

constexpr int P2P_STATUS = 128;  // p2p_sync words of rank 0 where rank r's frame status lands: [128 + 2r + parity] (R <= 127)

// ranks exchange keys with rank 0 (NCCL communicator or P2P buffers)
static bool exchanging(const piko_ctx* ctx) {
  return (ctx->comm != nullptr || ctx->p2p_keys != nullptr) && ctx->mnranks > 1;
}

static int p2p_export(piko_ctx* ctx, int nranks, void* h);
static int p2p_import(piko_ctx* ctx, const void* h, int rank, int nranks);
static_assert(2 * sizeof(cudaIpcMemHandle_t) <= PIKO_P2P_HANDLE_BYTES, "IPC handle bytes");

// rank 0: allocate the P2P exchange buffers (zeroed epochs)
static int p2p_alloc(piko_ctx* ctx) {
  const size_t tile = (size_t)ctx->bw * ctx->bh;
  const size_t nkeys = 2 * (size_t)ctx->mnranks * ctx->owned_max * tile;
  CK(cudaMalloc(&ctx->p2p_keys, sizeof(unsigned long long) * std::max<size_t>(nkeys, 1)));
  CK(cudaMalloc(&ctx->p2p_sync, 4096));
  CK(cudaMemset(ctx->p2p_sync, 0, 4096));
  ctx->p2p_owner = true;
  return PIKO_OK;
}

static void set_ownership(piko_ctx* ctx, int rank, int nranks) {
  ctx->mrank = rank;
  ctx->mnranks = nranks;
  if (ctx->multi == PIKO_MULTI_SORT_LAST) { rank = 0; nranks = 1; }  // every rank owns every bin
  ctx->g.rank = rank;
  ctx->g.nranks = nranks;
  ctx->owned = (int)piko_owned_bins(ctx->g.W, ctx->g.H, ctx->bw, ctx->bh, rank, nranks, nullptr, 0);
  ctx->owned_max = (int)piko_owned_bins(ctx->g.W, ctx->g.H, ctx->bw, ctx->bh, 0, nranks, nullptr, 0);
}

extern "C" piko_ctx* piko_create(int width, int height, int bin_w, int bin_h) {
  if (width < 1 || height < 1 || width > 16384 || height > 16384) {
    g_create_error = "width and height must be in [1, 16384]";
    return nullptr;
  }
  if (!pow2_in(bin_w, 8, 64) || !pow2_in(bin_h, 8, 64)) {
    g_create_error = "bin_w and bin_h must be powers of two in [8, 64]";
    return nullptr;
  }
  piko_ctx* ctx = new (std::nothrow) piko_ctx();
  if (!ctx) { g_create_error = "out of host memory"; return nullptr; }
  cudaGetDevice(&ctx->device);
  if (cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, ctx->device) != cudaSuccess || ctx->sms <= 0)
    ctx->sms = 148;
  ctx->bw = bin_w; ctx->bh = bin_h;
  Grid& g = ctx->g;
  g.W = width; g.H = height;
  g.bw_log2 = ilog2(bin_w); g.bh_log2 = ilog2(bin_h);
  g.binsX = (width + bin_w - 1) / bin_w;
  g.binsY = (height + bin_h - 1) / bin_h;
  g.NB = g.binsX * g.binsY;
  set_ownership(ctx, 0, 1);
  int bits = 0;
  while ((1ll << bits) < (long long)g.NB) ++bits;
  ctx->npass = std::max(1, (bits + RX_BITS - 1) / RX_BITS);  // pass 0 also expands the pairs
  const long long npx = (long long)width * height;
  bool ok = cudaMalloc(&ctx->bin_count, sizeof(uint32_t) * g.NB) == cudaSuccess &&
            cudaMalloc(&ctx->bin_start, sizeof(int32_t) * (g.NB + 1)) == cudaSuccess &&
            cudaMalloc(&ctx->bin_list, sizeof(int32_t) * (NLIST - 1) * (size_t)g.NB) == cudaSuccess &&
            cudaMalloc(&ctx->arrive, sizeof(uint32_t) * (size_t)g.NB) == cudaSuccess &&
            cudaMalloc(&ctx->ctl, sizeof(Control)) == cudaSuccess &&
            cudaMalloc(&ctx->primid, sizeof(int32_t) * npx) == cudaSuccess &&
            cudaMalloc(&ctx->sc.sink, 16) == cudaSuccess &&
            cudaMallocHost(&ctx->h_ctl, sizeof(Control)) == cudaSuccess;
  for (int k = 0; k < piko_ctx::NRING && ok; ++k)
    ok = cudaHostAlloc(&ctx->ring[k].h, sizeof(Control), cudaHostAllocMapped) == cudaSuccess &&
         cudaHostGetDevicePointer(&ctx->ring[k].d, ctx->ring[k].h, 0) == cudaSuccess &&
         cudaEventCreateWithFlags(&ctx->ring[k].ev, cudaEventDisableTiming) == cudaSuccess;
  ctx->st_scan_n = (g.NB + SCAN_CHUNK - 1) / SCAN_CHUNK;
  ok = ok && cudaMalloc(&ctx->st_scan, sizeof(unsigned long long) * ctx->st_scan_n) == cudaSuccess;
  ok = ok && cudaMemset(ctx->bin_count, 0, sizeof(uint32_t) * g.NB) == cudaSuccess &&
       cudaMemset(ctx->bin_start, 0, sizeof(int32_t) * (g.NB + 1)) == cudaSuccess &&
       cudaMemset(ctx->ctl, 0, sizeof(Control)) == cudaSuccess;
  if (!ok) {
    g_create_error = std::string("device allocation failed: ") + cudaGetErrorString(cudaGetLastError());
    piko_destroy(ctx);
    return nullptr;
  }
  memset(ctx->h_ctl, 0, sizeof(Control));
  if (const char* e = getenv("PIKO_NO_PDL")) ctx->pdl = e[0] == '0';
  if (const char* e = getenv("PIKO_SEPARATE_VS")) ctx->vs_mode = e[0] == '0' ? 0 : 1;
  if (const char* e = getenv("PIKO_DEFERRED")) ctx->deferred = e[0] == '0' ? 0 : 1;
  if (const char* e = getenv("PIKO_CM")) ctx->cm_mode = e[0] == '0' ? 0 : 1;
  if (const char* e = getenv("PIKO_CL")) ctx->cl_mode = e[0] == '0' ? 0 : 1;
  if (const char* e = getenv("PIKO_EARLY_EMPTY")) ctx->early_empty = e[0] == '0' ? 0 : 1;
  if (const char* e = getenv("PIKO_TILE_GRID")) ctx->tile_items_grid = strcmp(e, "items") == 0;
  if (const char* e = getenv("PIKO_CM_TC_LOG2")) ctx->cm_tc_log2 = atoi(e);
  return ctx;
}

extern "C" void piko_destroy(piko_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  for (int k = 0; k < ctx->ring_n; ++k)  // this context's frames in flight (not the whole device)
    cudaEventSynchronize(ctx->ring[(ctx->ring_head - ctx->ring_n + k + piko_ctx::NRING) % piko_ctx::NRING].ev);
  if (ctx->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(ctx->comm);
  if (ctx->p2p_ipc) {
    cudaIpcCloseMemHandle(ctx->p2p_keys);
    cudaIpcCloseMemHandle(ctx->p2p_sync);
  } else if (ctx->p2p_owner) {
    cudaFree(ctx->p2p_keys);
    cudaFree(ctx->p2p_sync);
  }
  void* bufs[] = {ctx->xv, ctx->rec, ctx->keys[0], ctx->keys[1], ctx->vals[0], ctx->vals[1], ctx->bin_count,
                  ctx->bin_start, ctx->frag_list, ctx->bin_list, ctx->fkey, ctx->gcov, ctx->arrive, ctx->ctl, ctx->rect, ctx->st_scan, ctx->st_rx, ctx->st_grp, ctx->ccount, ctx->garr, ctx->primid,
                  ctx->cov, ctx->d_verts, ctx->d_idx, ctx->d_rgba, ctx->d_depth, ctx->tile_keys, ctx->def_keys, ctx->cm, ctx->cp, ctx->dice_verts, ctx->dice_idx, ctx->dice_rate, ctx->dice_base, ctx->dice_total,
                  ctx->all_keys, ctx->fp_keys, ctx->ovq, ctx->sc.sink, ctx->bl_keys, ctx->frag_key,
                  ctx->frag_px, ctx->frag_rgba, ctx->cl_ent, ctx->cl_bm, ctx->cl_tot};
  for (void* p : bufs)
    if (p) cudaFree(p);
  if (ctx->h_ctl) cudaFreeHost(ctx->h_ctl);
  if (ctx->h_dice_total) cudaFreeHost(ctx->h_dice_total);
  for (auto& sl : ctx->ring) {
    if (sl.h) cudaFreeHost(sl.h);  // (cudaHostAlloc'ed)
    if (sl.ev) cudaEventDestroy(sl.ev);
  }
  for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
  for (auto& h : ctx->hs) {
    if (h.out_done) cudaEventSynchronize(h.out_done);
    void* hb[] = {h.verts, h.idx, h.rgba, h.depth};
    for (void* p : hb)
      if (p) cudaFree(p);
    for (cudaEvent_t e : {h.in_done, h.frame_done, h.out_done})
      if (e) cudaEventDestroy(e);
  }
  if (ctx->cs_in) cudaStreamDestroy(ctx->cs_in);
  if (ctx->cs_out) cudaStreamDestroy(ctx->cs_out);
  delete ctx;
}

extern "C" const char* piko_last_error(const piko_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_create_error.c_str();
}

// ---- capacity management ----------------------------------------------------
static int alloc_rx_status(piko_ctx* ctx);

static int ensure_tris(piko_ctx* ctx, long long T) {
  if (T > ctx->rec_cap) {
    long long cap = std::max<long long>(T, 1024);
    if (ctx->rec) cudaFree(ctx->rec);
    if (ctx->rect) cudaFree(ctx->rect);
    ctx->rec = nullptr;
    ctx->rect = nullptr;
    CK(cudaMalloc(&ctx->rec, sizeof(int4) * 3 * cap));
    CK(cudaMalloc(&ctx->rect, sizeof(uint2) * cap));
    ctx->rec_cap = cap;
    return alloc_rx_status(ctx);
  }
  return PIKO_OK;
}

// look-back status words: enough chunks for the expand pass (>= 256 triangles
// per chunk) and for the pair passes
static long long rx_slots(const piko_ctx* ctx) {  // radix CTAs resident at once
  return (long long)RX_MIN_CTAS * ctx->sms;
}

static int alloc_rx_status(piko_ctx* ctx) {
  const long long chunks = std::max<long long>(
      std::max<long long>((ctx->rec_cap + RX_THREADS - 1) / RX_THREADS,
                          (long long)((ctx->pair_cap + RX_CHUNK - 1) / RX_CHUNK)), 1);
  if (chunks > ctx->st_rx_chunks) {
    for (void* p : {(void*)ctx->st_rx, (void*)ctx->st_grp, (void*)ctx->ccount, (void*)ctx->garr})
      if (p) cudaFree(p);
    ctx->st_rx = nullptr; ctx->st_grp = nullptr; ctx->ccount = nullptr; ctx->garr = nullptr;
    const long long groups = (chunks + LB_GROUP - 1) / LB_GROUP;
    CK(cudaMalloc(&ctx->st_rx, sizeof(unsigned long long) * RX_RADIX * chunks * ctx->npass));
    CK(cudaMalloc(&ctx->ccount, sizeof(uint32_t) * RX_RADIX * chunks * ctx->npass));
    CK(cudaMalloc(&ctx->st_grp, sizeof(unsigned long long) * RX_RADIX * groups * ctx->npass));
    CK(cudaMalloc(&ctx->garr, sizeof(uint32_t) * 2 * groups * ctx->npass));
    ctx->st_rx_chunks = chunks;
    ctx->gcap = groups;
    ctx->need_reset = true;
  }
  return PIKO_OK;
}

static int ensure_pairs(piko_ctx* ctx, unsigned long long P) {
  if (P <= ctx->pair_cap) return PIKO_OK;
  if (P >= MAX_PAIRS)
    return ctx->fail(PIKO_ECAPACITY, "pair count %llu exceeds the 2^31 limit", P);
  unsigned long long cap = std::min<unsigned long long>(P + P / 4 + 4096, MAX_PAIRS - 1);
  for (int k = 0; k < 2; ++k) {
    if (ctx->keys[k]) cudaFree(ctx->keys[k]);
    if (ctx->vals[k]) cudaFree(ctx->vals[k]);
    ctx->keys[k] = nullptr; ctx->vals[k] = nullptr;
    CK(cudaMalloc(&ctx->keys[k], sizeof(uint32_t) * cap));
    CK(cudaMalloc(&ctx->vals[k], sizeof(int32_t) * cap));
  }
  ctx->pair_cap = cap;
  if (alloc_rx_status(ctx) != PIKO_OK) return PIKO_ECUDA;
  const long long fcap = (long long)(cap / (unsigned long long)tile_frag(ctx->bw, ctx->bh)) + ctx->g.NB + 1;
  if (ctx->frag_list) cudaFree(ctx->frag_list);
  ctx->frag_list = nullptr;
  CK(cudaMalloc(&ctx->frag_list, sizeof(int2) * fcap));
  if (ctx->fkey) cudaFree(ctx->fkey);
  ctx->fkey = nullptr;
  CK(cudaMalloc(&ctx->fkey, sizeof(unsigned long long) * (size_t)fcap * ctx->bw * ctx->bh));
  ctx->frag_cap = fcap;
  ctx->need_reset = true;
  return PIKO_OK;
}

// Vertex stage placement.  Separate (k_vertex: each vertex transformed once,
// 16 B records gathered by k_setup) wins on meshes whose vertices are shared by
// several triangles; fused (k_setup transforms its three corners from the raw
// 32 B vertices) wins when vertices are barely shared (soups: V ~ 3T) and for
// piko_draw without a vertex count (no k_index_max + k_vertex launches).
static bool separate_vs(const piko_ctx* ctx, long long V, long long T) {
  if (ctx->pipeline == PIKO_PIPE_BASELINE) return true;  // VS is its own stage
  if (ctx->vs_mode >= 0) return ctx->vs_mode == 1;
  if (V >= 0) return 2 * V <= 3 * T;
  // piko_draw (no vertex count): the separate stage would first derive V with
  // a k_index_max pass over idx and then need k_vertex -- two launches on the
  // critical path; the fused k_setup transforms the corners itself and is
  // faster on every mesh measured (c3 84 vs 88 us, c5 1262 vs 1336 us, c2
  // 163 vs 165 us)
  return false;
}

// xv capacity for V vertices (V < 0: unknown; sized from an upper bound)
static int ensure_verts(piko_ctx* ctx, long long V) {
  if (V > ctx->xv_cap) {
    if (ctx->xv) cudaFree(ctx->xv);
    ctx->xv = nullptr;
    CK(cudaMalloc(&ctx->xv, sizeof(int4) * std::max<long long>(V, 1024)));
    ctx->xv_cap = std::max<long long>(V, 1024);
  }
  return PIKO_OK;
}

static int ensure_cov(piko_ctx* ctx) {
  if ((ctx->debug & PIKO_DEBUG_COVERAGE_COUNT) && !ctx->cov) {
    CK(cudaMalloc(&ctx->cov, sizeof(uint32_t) * (size_t)ctx->g.W * ctx->g.H));
    CK(cudaMalloc(&ctx->gcov, sizeof(uint32_t) * (size_t)ctx->g.NB * ctx->bw * ctx->bh));
    ctx->need_reset = true;
  }
  return PIKO_OK;
}

// ---- frame status ring --------------------------------------------------------
static int eval_frame(piko_ctx* ctx, piko_ctx::Slot& sl);

// Evaluate finished frames in order; block only if `block` (all of them) --
// otherwise stop at the first frame still running.  Errors of async frames
// accumulate in ctx->sticky (the first one wins).
static int poll_frames(piko_ctx* ctx, bool block) {
  while (ctx->ring_n > 0) {
    piko_ctx::Slot& sl = ctx->ring[(ctx->ring_head - ctx->ring_n + piko_ctx::NRING) % piko_ctx::NRING];
    if (block) {
      CK(cudaEventSynchronize(sl.ev));
    } else {
      const cudaError_t q = cudaEventQuery(sl.ev);
      if (q == cudaErrorNotReady) break;
      if (q != cudaSuccess) CK(q);
    }
    --ctx->ring_n;
    const int rc = eval_frame(ctx, sl);
    if (rc != PIKO_OK && ctx->sticky == PIKO_OK) ctx->sticky = rc;
  }
  ctx->pending = ctx->ring_n > 0;
  return PIKO_OK;
}

// Make the next ring slot free (a full ring waits for its oldest frame) and
// return its mirror's device alias (the binned frame's tile kernel writes the
// control block into it: no copy on the stream).
static cudaError_t reserve_slot(piko_ctx* ctx, Control** dev_mirror) {
  if (ctx->ring_n == piko_ctx::NRING && poll_frames(ctx, false) == PIKO_OK && ctx->ring_n == piko_ctx::NRING) {
    piko_ctx::Slot& old = ctx->ring[ctx->ring_head];  // == oldest when full
    cudaError_t e = cudaEventSynchronize(old.ev);
    if (e != cudaSuccess) return e;
    --ctx->ring_n;
    const int rc = eval_frame(ctx, old);
    if (rc != PIKO_OK && ctx->sticky == PIKO_OK) ctx->sticky = rc;
  }
  if (dev_mirror) *dev_mirror = ctx->ring[ctx->ring_head].d;
  return cudaSuccess;
}

// Queue the end of a frame: its control block into the next ring slot's
// pinned mirror (unless the last kernel already wrote it) and an event.
static cudaError_t record_frame_end(piko_ctx* ctx, cudaStream_t s, long long T, bool mirrored = false) {
  cudaError_t e = reserve_slot(ctx, nullptr);
  if (e != cudaSuccess) return e;
  piko_ctx::Slot& sl = ctx->ring[ctx->ring_head];
  if (!mirrored) e = cudaMemcpyAsync(sl.h, ctx->ctl, offsetof(Control, digit_hist), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaEventRecord(sl.ev, s);
  if (e != cudaSuccess) return e;
  sl.T = T;
  sl.cm = ctx->pipeline == PIKO_PIPE_BINNED && ctx->last_cm;
  ctx->ring_head = (ctx->ring_head + 1) % piko_ctx::NRING;
  ++ctx->ring_n;
  ctx->pending = true;
  return cudaSuccess;
}

// ---- one frame ---------------------------------------------------------------
static int enqueue_freepipe(piko_ctx* ctx, const float* verts, long long V, const int32_t* idx,
                            long long T, const Mat4& M, const float L[3], float* rgba, float* depth,
                            cudaStream_t s) {
  cudaEvent_t* ev = ctx->prof ? ctx->frame_events() : nullptr;
  auto mark = [&](int stage) -> cudaError_t { return ev ? cudaEventRecord(ev[stage], s) : cudaSuccess; };
  const size_t npx = (size_t)ctx->g.W * ctx->g.H;
  CK(mark(0));
  if (!ctx->fp_keys) {
    CK(cudaMalloc(&ctx->fp_keys, sizeof(unsigned long long) * npx));
    CK(cudaMemsetAsync(ctx->fp_keys, 0xFF, sizeof(unsigned long long) * npx, s));
  }
  if (ctx->debug & PIKO_DEBUG_COVERAGE_COUNT) CK(cudaMemsetAsync(ctx->cov, 0, sizeof(uint32_t) * npx, s));
  // the control block is still used for the device vertex count
  CK(mark(1 + PIKO_STAGE_CLEAR));
  const bool sep = separate_vs(ctx, V, T);
  ctx->last_kernels = 2 + (T > 0 ? 1 : 0) + (sep && V < 0 && T > 0 ? 1 : 0);
  if (sep) {  // vmax and vx_overflow (adjacent) start at 0
    CK(cudaMemsetAsync(&ctx->ctl->vmax, 0, 2 * sizeof(unsigned), s));
    if (V < 0 && T > 0) CK(launch_index_max(idx, 3 * T, ctx->ctl, ctx->pdl, s));
    VertexArgs va{};
    va.verts = verts; va.n_verts = T > 0 ? V : 0; va.cap = ctx->xv_cap; va.ctl = ctx->ctl; va.M = M;
    va.W = ctx->g.W; va.H = ctx->g.H; va.xv = ctx->xv;
    CK(launch_vertex(va, ctx->pdl, s));
  }
  CK(mark(1 + PIKO_STAGE_VERTEX));
  FreePipeArgs a{};
  a.verts = verts; a.xv = sep ? ctx->xv : nullptr; a.xv_cap = ctx->xv_cap; a.M = M;
  a.idx = idx; a.n_tris = T;
  a.W = ctx->g.W; a.H = ctx->g.H; a.keys = ctx->fp_keys;
  a.cov = (ctx->debug & PIKO_DEBUG_COVERAGE_COUNT) ? ctx->cov : nullptr;
  a.light[0] = L[0]; a.light[1] = L[1]; a.light[2] = L[2];
  a.out_rgba = rgba; a.out_depth = depth; a.out_primid = ctx->primid;
  a.sc = ctx->sc;
  if (T > 0) CK(launch_freepipe(a, ctx->pdl, s));
  CK(mark(1 + PIKO_STAGE_SETUP));
  CK(mark(1 + PIKO_STAGE_EXPAND));
  CK(mark(1 + PIKO_STAGE_SORT));
  CK(launch_fp_resolve(a, ctx->pdl, s));
  CK(mark(1 + PIKO_STAGE_TILE));
  CK(mark(1 + PIKO_STAGE_GATHER));
  CK(mark(1 + PIKO_STAGE_RESOLVE));
  if (ev) ++ctx->prof_frames;
  // no pair capacity to check: report a clean frame to the host mirror, except
  // a vertex-capacity overflow of k_vertex (vx_overflow / vx_need kept)
  CK(cudaMemsetAsync(ctx->ctl, 0, offsetof(Control, vx_overflow), s));
  CK(cudaMemsetAsync(&ctx->ctl->n_pairs, 0, sizeof(unsigned long long) * 2, s));
  CK(record_frame_end(ctx, s, T));
  ctx->last_T = T;
  ctx->need_reset = true;  // the binned path must not trust tickets touched here
  return PIKO_OK;
}

// fragment buffers of the Baseline pipeline for n fragments
static int ensure_frags(piko_ctx* ctx, long long n) {
  if (n <= ctx->bl_cap) return PIKO_OK;
  cudaFree(ctx->frag_key); cudaFree(ctx->frag_px); cudaFree(ctx->frag_rgba);
  ctx->frag_key = nullptr; ctx->frag_px = nullptr; ctx->frag_rgba = nullptr; ctx->bl_cap = 0;
  const long long cap = std::max<long long>(n + n / 4, 1 << 16);
  CK(cudaMalloc(&ctx->frag_key, sizeof(unsigned long long) * cap));
  CK(cudaMalloc(&ctx->frag_px, sizeof(uint32_t) * cap));
  CK(cudaMalloc(&ctx->frag_rgba, sizeof(float4) * cap));
  ctx->bl_cap = cap;
  return PIKO_OK;
}

// Baseline: VS, Rasterizer, Fragment Shader, Depth Test,
// Composite as separate kernels with off-chip buffers between them.  Profiling
// stages: VERTEX = VS, SETUP = Rasterizer, EXPAND = Fragment Shader, SORT =
// Depth Test, TILE = Composite.  The fragment count is read back by
// check_frame; a frame that overflowed the buffers is grown and re-issued.
static int enqueue_baseline(piko_ctx* ctx, const float* verts, long long V, const int32_t* idx,
                            long long T, const Mat4& M, const float L[3], float* rgba, float* depth,
                            cudaStream_t s) {
  cudaEvent_t* ev = ctx->prof ? ctx->frame_events() : nullptr;
  auto mark = [&](int stage) -> cudaError_t { return ev ? cudaEventRecord(ev[stage], s) : cudaSuccess; };
  const size_t npx = (size_t)ctx->g.W * ctx->g.H;
  CK(mark(0));
  if (!ctx->bl_keys) {
    CK(cudaMalloc(&ctx->bl_keys, sizeof(unsigned long long) * npx));
    CK(cudaMemsetAsync(ctx->bl_keys, 0xFF, sizeof(unsigned long long) * npx, s));
  }
  int rc = ensure_frags(ctx, std::max<long long>(4ll * (long long)npx, 2 * T));
  if (rc != PIKO_OK) return rc;
  if (ctx->debug & PIKO_DEBUG_COVERAGE_COUNT) CK(cudaMemsetAsync(ctx->cov, 0, sizeof(uint32_t) * npx, s));
  // clean control block (the fragment count lives in n_pairs)
  CK(cudaMemsetAsync(ctx->ctl, 0, offsetof(Control, vx_overflow), s));
  CK(cudaMemsetAsync(&ctx->ctl->n_pairs, 0, sizeof(unsigned long long) * 2, s));
  CK(mark(1 + PIKO_STAGE_CLEAR));
  ctx->last_kernels = 6 + (V < 0 && T > 0 ? 1 : 0);
  CK(cudaMemsetAsync(&ctx->ctl->vmax, 0, 2 * sizeof(unsigned), s));
  if (V < 0 && T > 0) CK(launch_index_max(idx, 3 * T, ctx->ctl, ctx->pdl, s));
  VertexArgs va{};
  va.verts = verts; va.n_verts = T > 0 ? V : 0; va.cap = ctx->xv_cap; va.ctl = ctx->ctl; va.M = M;
  va.W = ctx->g.W; va.H = ctx->g.H; va.xv = ctx->xv;
  CK(launch_vertex(va, ctx->pdl, s));
  CK(mark(1 + PIKO_STAGE_VERTEX));
  BaselineArgs a{};
  a.verts = verts; a.xv = ctx->xv; a.xv_cap = ctx->xv_cap; a.M = M; a.idx = idx; a.n_tris = T;
  a.W = ctx->g.W; a.H = ctx->g.H;
  a.light[0] = L[0]; a.light[1] = L[1]; a.light[2] = L[2];
  a.keys = ctx->bl_keys; a.frag_key = ctx->frag_key; a.frag_px = ctx->frag_px;
  a.frag_rgba = ctx->frag_rgba; a.frag_cap = ctx->bl_cap; a.n_frag = &ctx->ctl->n_pairs;
  a.cov = (ctx->debug & PIKO_DEBUG_COVERAGE_COUNT) ? ctx->cov : nullptr;
  a.out_rgba = rgba; a.out_depth = depth; a.out_primid = ctx->primid;
  a.sc = ctx->sc;
  CK(launch_baseline(a, 0, ctx->pdl, s));
  CK(mark(1 + PIKO_STAGE_SETUP));
  CK(launch_baseline(a, 1, ctx->pdl, s));
  CK(mark(1 + PIKO_STAGE_EXPAND));
  CK(launch_baseline(a, 2, ctx->pdl, s));
  CK(mark(1 + PIKO_STAGE_SORT));
  CK(launch_baseline(a, 3, ctx->pdl, s));
  CK(launch_baseline(a, 4, ctx->pdl, s));
  CK(mark(1 + PIKO_STAGE_TILE));
  CK(mark(1 + PIKO_STAGE_GATHER));
  CK(mark(1 + PIKO_STAGE_RESOLVE));
  if (ev) ++ctx->prof_frames;
  CK(record_frame_end(ctx, s, T));
  ctx->last_T = T;
  ctx->need_reset = true;  // the binned path must not trust tickets touched here
  return PIKO_OK;
}

// Count-matrix AssignBin for this frame?  Rows of 2^cm_shift triangles (a
// multiple of K1_CHUNK): enough rows for about two resident scatter CTAs per
// SM, fewer (longer) rows when rows x NB would exceed CM_MAX_ENTRIES.
static bool use_cm(const piko_ctx* ctx, long long T, int& shift, long long& rows) {
  if (ctx->cm_mode == 0 || ctx->npass < 1 || ctx->g.NB > CM_MAX_NB) return false;
  // a count-matrix frame of this size showed dense rows (most of a window's
  // pairs in distinct bins: an unordered soup) -- the radix passes rank those
  // with less work (c4: 1179 vs 1139 us); auto mode only
  if (ctx->cm_mode < 0 && ctx->cm_dense_T == T) return false;
  shift = 10;  // K1_CHUNK
  if (ctx->cm_tc_log2 >= 10) shift = ctx->cm_tc_log2;
  else
    while ((T >> shift) > 2ll * ctx->sms) ++shift;
  rows = std::max<long long>((T + (1ll << shift) - 1) >> shift, 1);
  while (rows * ctx->g.NB > CM_MAX_ENTRIES && shift < 30) {
    ++shift;
    rows = std::max<long long>((T + (1ll << shift) - 1) >> shift, 1);
  }
  return rows * ctx->g.NB <= CM_MAX_ENTRIES;
}

static int ensure_cm(piko_ctx* ctx, long long rows) {
  const long long need = rows * ctx->g.NB;
  if (need > ctx->cm_cap) {
    if (ctx->cm) cudaFree(ctx->cm);
    if (ctx->cp) cudaFree(ctx->cp);
    ctx->cm = nullptr; ctx->cp = nullptr; ctx->cm_cap = 0;
    CK(cudaMalloc(&ctx->cm, sizeof(uint32_t) * need));
    CK(cudaMalloc(&ctx->cp, sizeof(uint32_t) * need));
    ctx->cm_cap = need;
    ctx->need_reset = true;  // the matrix is zeroed by the reset
  }
  return PIKO_OK;
}

// Chunk-list AssignBin for this frame?  k_setup CTAs (chunks of K1_CHUNK
// triangles) record per bin the mask of their 32-triangle groups with a pair
// in it (per-bin arrays in shared memory: NB <= CL_MAX_NB) and k_cl_bins
// compacts every bin's candidates; off after a bin had more than CLB_ENT
// chunks or CLB_GRP groups (unordered soups: the count matrix handles them).
static bool use_cl(const piko_ctx* ctx, long long T, long long& nch, int& nw) {
  nch = (T + K1_CHUNK - 1) / K1_CHUNK;
  nw = (int)((nch + 31) / 32);
  if (ctx->cl_mode == 0 || ctx->cl_off || T <= 0 || ctx->g.NB > CL_MAX_NB) return false;
  return nw <= CLB_THREADS * CL_WPT && nch * ctx->g.NB <= CL_MAX_ENTRIES;
}

static int ensure_cl(piko_ctx* ctx, long long nch, int nw) {
  const long long NB = ctx->g.NB;
  if (NB * nch > ctx->cl_ent_cap) {
    if (ctx->cl_ent) cudaFree(ctx->cl_ent);
    ctx->cl_ent = nullptr; ctx->cl_ent_cap = 0;
    CK(cudaMalloc(&ctx->cl_ent, sizeof(uint2) * NB * nch));
    ctx->cl_ent_cap = NB * nch;
  }
  if (NB * nw > ctx->cl_bm_cap) {
    if (ctx->cl_bm) cudaFree(ctx->cl_bm);
    ctx->cl_bm = nullptr; ctx->cl_bm_cap = 0;
    CK(cudaMalloc(&ctx->cl_bm, sizeof(uint32_t) * NB * nw));
    ctx->cl_bm_cap = NB * nw;
    ctx->need_reset = true;  // bitmaps are zeroed by the reset
  }
  if (!ctx->cl_tot) {
    CK(cudaMalloc(&ctx->cl_tot, sizeof(uint32_t) * 2 * NB));
    ctx->need_reset = true;
  }
  return PIKO_OK;
}

static int enqueue_frame(piko_ctx* ctx, const float* verts, long long V, const int32_t* idx,
                         long long T, const Mat4& M, const float L[3], float* rgba, float* depth,
                         cudaStream_t s, unsigned long long* keys_out = nullptr) {
  if (ctx->pipeline == PIKO_PIPE_FREEPIPE)
    return enqueue_freepipe(ctx, verts, V, idx, T, M, L, rgba, depth, s);
  if (ctx->pipeline == PIKO_PIPE_BASELINE)
    return enqueue_baseline(ctx, verts, V, idx, T, M, L, rgba, depth, s);
  const bool gather = keys_out == nullptr && exchanging(ctx);
  const bool p2p = gather && ctx->p2p_keys != nullptr;
  const size_t tile_px = (size_t)ctx->bw * ctx->bh;
  if (p2p) ++ctx->epoch;
  // P2P: this frame's key slot (epoch parity) at rank 0
  unsigned long long* p2p_slot = p2p ? ctx->p2p_keys + (size_t)(ctx->epoch & 1) * ctx->mnranks * ctx->owned_max * tile_px
                                     : nullptr;
  // single GPU, no debug coverage: keys-only tile kernel + k_resolve
  const bool defer = !gather && keys_out == nullptr && ctx->deferred && ctx->mnranks == 1 &&
                     !(ctx->debug & PIKO_DEBUG_COVERAGE_COUNT);
  if (defer && !ctx->def_keys)
    CK(cudaMalloc(&ctx->def_keys, sizeof(unsigned long long) * (size_t)ctx->g.NB * tile_px));
  const bool keys_only = gather || keys_out != nullptr || defer;
  cudaEvent_t* ev = ctx->prof ? ctx->frame_events() : nullptr;
  if (ctx->prof && !ev) return ctx->fail(PIKO_ECUDA, "cannot create profiling events");
  auto mark = [&](int stage) -> cudaError_t { return ev ? cudaEventRecord(ev[stage], s) : cudaSuccess; };
  const long long g1 = std::max<long long>((T + K1_CHUNK - 1) / K1_CHUNK, 1);
  const long long ntiles = (ctx->g.NB + SCAN_CHUNK - 1) / SCAN_CHUNK;
  const long long gx = std::max<long long>((T + ctx->tri_chunk - 1) / ctx->tri_chunk, 1);  // pass 0
  const long long gp = (long long)((ctx->pair_cap + RX_CHUNK - 1) / RX_CHUNK);              // passes >= 1
  int cm_shift = 0, cl_nw = 0;
  long long cm_rows = 0, cl_nch = 0;
  const bool clm = use_cl(ctx, T, cl_nch, cl_nw);
  if (clm && ensure_cl(ctx, cl_nch, cl_nw) != PIKO_OK) return PIKO_ECUDA;
  const bool cm = !clm && use_cm(ctx, T, cm_shift, cm_rows);
  if (cm && ensure_cm(ctx, cm_rows) != PIKO_OK) return PIKO_ECUDA;
  const bool sorted_here = cm || clm;  // no radix passes this frame
  const long long grids[6] = {g1, gx, gp + ntiles, ntiles, clm ? 2 : cm ? 1 : 0, cm ? cm_rows : 0};
  CK(mark(0));
  bool changed = ctx->need_reset;
  for (int k = 0; k < 6; ++k) changed |= grids[k] != ctx->last_grids[k];
  if (changed) {
    if (ctx->cm) CK(cudaMemsetAsync(ctx->cm, 0, sizeof(uint32_t) * ctx->cm_cap, s));
    if (ctx->cl_bm) CK(cudaMemsetAsync(ctx->cl_bm, 0, sizeof(uint32_t) * ctx->cl_bm_cap, s));
    if (ctx->cl_tot) CK(cudaMemsetAsync(ctx->cl_tot, 0, sizeof(uint32_t) * 2 * ctx->g.NB, s));
    // tickets restart at 0, so every tag-carrying status word must be cleared
    CK(cudaMemsetAsync(ctx->ctl, 0, sizeof(Control), s));
    CK(cudaMemsetAsync(ctx->st_scan, 0, sizeof(unsigned long long) * ctx->st_scan_n, s));
    CK(cudaMemsetAsync(ctx->st_rx, 0, sizeof(unsigned long long) * RX_RADIX * ctx->st_rx_chunks * ctx->npass, s));
    CK(cudaMemsetAsync(ctx->st_grp, 0, sizeof(unsigned long long) * RX_RADIX * ctx->gcap * ctx->npass, s));
    CK(cudaMemsetAsync(ctx->garr, 0, sizeof(uint32_t) * 2 * ctx->gcap * ctx->npass, s));
    CK(cudaMemsetAsync(ctx->bin_count, 0, sizeof(uint32_t) * ctx->g.NB, s));
    CK(cudaMemsetAsync(ctx->arrive, 0, sizeof(uint32_t) * ctx->g.NB, s));
    if (ctx->gcov) CK(cudaMemsetAsync(ctx->gcov, 0, sizeof(uint32_t) * ctx->g.NB * ctx->bw * ctx->bh, s));
    for (int k = 0; k < 6; ++k) ctx->last_grids[k] = grids[k];
    ctx->need_reset = false;
    ctx->frames = 0;
  }
  CK(mark(1 + PIKO_STAGE_CLEAR));
  const bool sep = separate_vs(ctx, V, T);
  ctx->last_kernels = 2 + (clm ? 1 : cm ? 2 : ctx->npass + (ctx->npass == 1 ? 1 : 0)) +
                      (sep ? 1 + (V < 0 && T > 0 ? 1 : 0) : 0) + (gather && ctx->mrank == 0 ? 1 : 0) + (defer ? 1 : 0);
  if (sep) {
    if (V < 0 && T > 0) CK(launch_index_max(idx, 3 * T, ctx->ctl, ctx->pdl, s));
    VertexArgs a{};
    a.verts = verts; a.n_verts = T > 0 ? V : 0; a.cap = ctx->xv_cap; a.ctl = ctx->ctl; a.M = M;
    a.W = ctx->g.W; a.H = ctx->g.H; a.xv = ctx->xv;
    CK(launch_vertex(a, ctx->pdl, s));
  }
  CK(mark(1 + PIKO_STAGE_VERTEX));
  {
    SetupArgs a{};
    a.xv = sep ? ctx->xv : nullptr; a.xv_cap = ctx->xv_cap; a.verts = verts; a.M = M;
    a.idx = idx; a.n_tris = T; a.g = ctx->g;
    a.npass = sorted_here ? 0 : ctx->npass; a.rec = ctx->rec; a.rec_stride = ctx->rec_cap; a.rect = ctx->rect; a.ctl = ctx->ctl;
    a.cm = cm ? ctx->cm : nullptr; a.cm_shift = cm_shift;
    a.frame = ctx->frames++;
    if (clm) {
      a.cl_ent = ctx->cl_ent; a.cl_bm = ctx->cl_bm;
      a.cl_tot = ctx->cl_tot + (size_t)(a.frame & 1) * ctx->g.NB;
      a.cl_nch = cl_nch; a.cl_nw = cl_nw;
      a.cl_start = ctx->bin_start; a.cl_cap = ctx->pair_cap;
    }
    CK(launch_setup(a, (int)g1, ctx->pdl, s));
  }
  CK(mark(1 + PIKO_STAGE_SETUP));
  ctx->prims_out = sorted_here ? ctx->vals[0] : ctx->vals[ctx->npass & 1];
  ctx->last_cm = cm;
  ctx->last_cm_rows = cm ? cm_rows : 0;
  ctx->last_cl = clm;
  ctx->last_cl_nch = clm ? cl_nch : 0;
  for (int p = 0; p < (sorted_here ? 0 : ctx->npass); ++p) {
    RadixArgs a{};
    a.expand = p == 0; a.rect = ctx->rect; a.n_tris = T; a.tri_chunk = ctx->tri_chunk;
    a.g = ctx->g; a.cap = ctx->pair_cap; a.scan_here = p == 1;
    a.keys_in = ctx->keys[p & 1]; a.vals_in = ctx->vals[p & 1];
    a.keys_out = (p + 1 < ctx->npass) ? ctx->keys[(p + 1) & 1] : nullptr;
    a.vals_out = ctx->vals[(p + 1) & 1];
    a.status = ctx->st_rx + (size_t)p * RX_RADIX * ctx->st_rx_chunks;
    a.ccount = ctx->ccount + (size_t)p * RX_RADIX * ctx->st_rx_chunks;
    a.gstatus = ctx->st_grp + (size_t)p * RX_RADIX * ctx->gcap;
    a.garrive = ctx->garr + (size_t)p * 2 * ctx->gcap;
    a.gcap = ctx->gcap;
    a.ctl = ctx->ctl; a.pass = p; a.shift = RX_BITS * p;
    a.bin_count = ctx->bin_count; a.bin_start = ctx->bin_start; a.scan_status = ctx->st_scan;
    a.NB = ctx->g.NB; a.rank = ctx->g.rank; a.nranks = ctx->g.nranks;
    a.frag_list = ctx->frag_list; a.bin_list = ctx->bin_list;
    a.gcov = (ctx->debug & PIKO_DEBUG_COVERAGE_COUNT) ? ctx->gcov : nullptr;
    a.frag = tile_frag(ctx->bw, ctx->bh); a.npx = ctx->bw * ctx->bh;
    CK(launch_radix_pass(a, (int)(p == 0 ? gx : gp + (p == 1 ? ntiles : 0)), ctx->pdl, s));
    if (p == 0 && ctx->npass == 1) CK(launch_bin_scan(a, (int)ntiles, ctx->pdl, s));
    if (p == 0) CK(mark(1 + PIKO_STAGE_EXPAND));
  }
  if (cm) {
    CmArgs c{};
    c.cm = ctx->cm; c.cp = ctx->cp; c.rows = cm_rows; c.cm_shift = cm_shift;
    c.rect = ctx->rect; c.n_tris = T; c.g = ctx->g; c.cap = ctx->pair_cap; c.bin_prims = ctx->prims_out;
    c.ctl = ctx->ctl;
    RadixArgs& a = c.sched;
    a.g = ctx->g; a.ctl = ctx->ctl; a.bin_start = ctx->bin_start; a.bin_count = ctx->bin_count; a.NB = ctx->g.NB;
    a.rank = ctx->g.rank; a.nranks = ctx->g.nranks;
    a.frag_list = ctx->frag_list; a.bin_list = ctx->bin_list;
    a.frag = tile_frag(ctx->bw, ctx->bh); a.npx = ctx->bw * ctx->bh;
    CK(launch_cm_scan(c, cm_scan_grid(ctx->g.NB), ctx->pdl, s));
    CK(mark(1 + PIKO_STAGE_EXPAND));
    CK(launch_cm_scatter(c, (int)(cm_rows + ntiles), ctx->pdl, s));
  }
  if (clm) {
    ClArgs c{};
    c.cl_ent = ctx->cl_ent; c.rect = ctx->rect; c.n_tris = T; c.cl_bm = ctx->cl_bm; c.cl_tot = ctx->cl_tot;
    c.nch = cl_nch; c.nw = cl_nw; c.frame = ctx->frames - 1;
    // persistent: CTA j owns bins j + k * grid (<= CLB_KMAX each)
    c.nbin_ctas = std::min(ctx->g.NB, std::max(8 * ctx->sms, (ctx->g.NB + CLB_KMAX - 1) / CLB_KMAX));
    c.g = ctx->g; c.cap = ctx->pair_cap; c.bin_prims = ctx->prims_out; c.ctl = ctx->ctl;
    RadixArgs& a = c.sched;
    a.g = ctx->g; a.ctl = ctx->ctl; a.bin_start = ctx->bin_start; a.bin_count = ctx->bin_count; a.NB = ctx->g.NB;
    a.rank = ctx->g.rank; a.nranks = ctx->g.nranks;
    a.frag_list = ctx->frag_list; a.bin_list = ctx->bin_list;
    a.frag = tile_frag(ctx->bw, ctx->bh); a.npx = ctx->bw * ctx->bh;
    CK(mark(1 + PIKO_STAGE_EXPAND));
    CK(launch_cl_bins(c, (int)(c.nbin_ctas + ntiles), ctx->pdl, s));
  }
  if (ctx->npass == 0) CK(mark(1 + PIKO_STAGE_EXPAND));
  CK(mark(1 + PIKO_STAGE_SORT));
  {
    TileArgs a{};
    a.sc = ctx->sc;
    a.verts = verts; a.xv = sep ? ctx->xv : nullptr; a.M = M; a.idx = idx;
    a.light[0] = L[0]; a.light[1] = L[1]; a.light[2] = L[2];
    a.g = ctx->g; a.npass = ctx->npass; a.rec = ctx->rec; a.rec_stride = ctx->rec_cap; a.bin_start = ctx->bin_start;
    a.bin_prims = ctx->prims_out; a.ctl = ctx->ctl;
    a.out_rgba = rgba; a.out_depth = depth; a.out_primid = ctx->primid;
    a.out_cov = (ctx->debug & PIKO_DEBUG_COVERAGE_COUNT) ? ctx->cov : nullptr;
    a.tile_keys = keys_out ? keys_out
                : p2p    ? p2p_slot + (size_t)ctx->mrank * ctx->owned_max * tile_px
                : gather ? ctx->tile_keys
                : defer  ? ctx->def_keys : nullptr;
    if (p2p) {
      a.p2p_flag = ctx->p2p_sync + ctx->mrank;
      a.p2p_done = ctx->p2p_sync + ctx->mnranks;
      a.epoch = ctx->epoch;
      // by epoch parity, like the key slots: a rank may run one frame ahead
      a.status_word = ctx->p2p_sync + P2P_STATUS + 2 * ctx->mrank + (ctx->epoch & 1);  // ok: the epoch
      a.status_ok = ctx->epoch;
    } else if (gather) {
      a.status_word = ctx->tile_keys + (size_t)ctx->owned_max * tile_px;
      a.status_ok = 1;
    }
    a.owned = ctx->owned;
    a.frag_list = ctx->frag_list; a.bin_list = ctx->bin_list;
    a.fkey = ctx->fkey; a.gcov = ctx->gcov; a.arrive = ctx->arrive; a.frag = tile_frag(ctx->bw, ctx->bh);
    a.garrive = ctx->garr; a.gcap = ctx->gcap;
    a.prim_base = (unsigned)ctx->prim_base;
    a.radix = sorted_here ? 0 : 1;
    a.skip_empty = defer && ctx->g.NB > 1 ? 1 : 0;
    // the counts are final two launches before k_tile in count-matrix frames
    a.early_empty = cm && !keys_only && ctx->early_empty ? 1 : 0;
    a.bin_count = ctx->bin_count;
    if (!gather) CK(reserve_slot(ctx, &a.status_out));  // the tile kernel ends the frame's control updates
    if (keys_only) a.out_cov = nullptr;
    // persistent grid (all CTAs resident, items from the queue) or, with
    // PIKO_TILE_GRID=items, one CTA per possible work item so the hardware
    // block scheduler balances them (the paper's LoadBalance)
    const int pers = std::max(1, std::min(ctx->owned, tile_grid(ctx->bw, ctx->bh, a.out_cov != nullptr, keys_only)));
    const int grid = ctx->tile_items_grid ? (int)std::max<long long>(pers, std::min<long long>(ctx->owned + ctx->frag_cap, INT32_MAX / 2))
                                          : pers;
    if (pers > ctx->ovq_ctas) {  // spill space of the per-bin large-triangle queue (per resident CTA)
      if (ctx->ovq) cudaFree(ctx->ovq);
      ctx->ovq = nullptr;
      ctx->ovq_ctas = 0;
      CK(cudaMalloc(&ctx->ovq, sizeof(int4) * 6 * OVQ_CAP * (size_t)pers));
      ctx->ovq_ctas = pers;
    }
    a.ovq = grid == pers ? ctx->ovq : nullptr;  // item grid: overflow takes the warp-cooperative path
    CK(launch_tile(a, ctx->bw, ctx->bh, grid, a.out_cov != nullptr, keys_only, ctx->pdl, s));
  }
  CK(mark(1 + PIKO_STAGE_TILE));
  if (gather) {
    const size_t tile_bytes = sizeof(unsigned long long) * ctx->bw * ctx->bh;
    const size_t bytes = tile_bytes * ctx->owned_max;
    int rc = 0;
    if (p2p) {
      // keys already at rank 0 (stored by k_tile over NVLink); nothing to send
    } else if (ctx->multi == PIKO_MULTI_SORT_LAST) {
      // element-wise (depth, primID) minimum of the full key images on rank 0
      // (+ the status word: the minimum is 0 if any rank overflowed)
      rc = g_nccl.Reduce(ctx->tile_keys, ctx->mrank == 0 ? ctx->all_keys : nullptr,
                         (size_t)ctx->owned * ctx->bw * ctx->bh + 1, ncclUint64_, ncclMin_, 0, ctx->comm, s);
      if (rc != 0) return ctx->fail(PIKO_ENCCL, "ncclReduce failed: %s", g_nccl.GetErrorString(rc));
    } else {
    if (g_nccl.GroupStart() != 0) return ctx->fail(PIKO_ENCCL, "ncclGroupStart failed");
    if (ctx->g.rank == 0) {
      // every rank's block is owned_max tiles + its status word
      const size_t blk = sizeof(unsigned long long) * ((size_t)ctx->owned_max * tile_px + 1);
      CK(cudaMemcpyAsync(ctx->all_keys, ctx->tile_keys, blk, cudaMemcpyDeviceToDevice, s));
      for (int r = 1; r < ctx->g.nranks && rc == 0; ++r)
        rc = g_nccl.Recv(reinterpret_cast<unsigned char*>(ctx->all_keys) + (size_t)r * blk, blk, ncclUint8_, r,
                         ctx->comm, s);
    } else {
      rc = g_nccl.Send(ctx->tile_keys, sizeof(unsigned long long) * ((size_t)ctx->owned_max * tile_px + 1),
                       ncclUint8_, 0, ctx->comm, s);
    }
    const int rc2 = g_nccl.GroupEnd();
    if (rc != 0 || rc2 != 0)
      return ctx->fail(PIKO_ENCCL, "NCCL gather failed: %s", g_nccl.GetErrorString(rc ? rc : rc2));
    }
    (void)bytes;
    CK(mark(1 + PIKO_STAGE_GATHER));
    if (ctx->mrank == 0) {
      // winners may come from any rank's triangles: re-transform their corners
      // from verts (xv may cover only this rank's range) with the full idx
      ResolveArgs a{};
      a.verts = verts; a.xv = nullptr; a.M = M; a.idx = idx - 3 * ctx->prim_base;
      a.light[0] = L[0]; a.light[1] = L[1]; a.light[2] = L[2];
      a.g = ctx->g; a.all_keys = ctx->all_keys; a.owned_max = ctx->owned_max;
      a.out_rgba = rgba; a.out_depth = depth; a.out_primid = ctx->primid;
      a.ctl = ctx->ctl;
      if (p2p) {
        a.all_keys = p2p_slot;
        a.p2p_flags = ctx->p2p_sync;
        a.p2p_done = ctx->p2p_sync + ctx->mnranks;
        a.p2p_count = &ctx->ctl->p2p_count;
        a.p2p_timeout = &ctx->ctl->p2p_timeout;
        a.epoch = ctx->epoch;
        a.status = ctx->p2p_sync + P2P_STATUS + (ctx->epoch & 1); a.status_stride = 2; a.nstatus = ctx->mnranks;
        a.status_ok = ctx->epoch;
      } else if (ctx->multi == PIKO_MULTI_SORT_LAST) {
        a.status = ctx->all_keys + (size_t)ctx->owned * tile_px; a.nstatus = 1; a.status_ok = 1;
      } else {
        a.rank_stride = (long long)ctx->owned_max * tile_px + 1;
        a.status = ctx->all_keys + (size_t)ctx->owned_max * tile_px;
        a.status_stride = a.rank_stride; a.nstatus = ctx->mnranks; a.status_ok = 1;
      }
      CK(launch_resolve(a, false, s));
    }
  } else {
    CK(mark(1 + PIKO_STAGE_GATHER));
    if (defer) {
      ResolveArgs a{};
      a.verts = verts; a.xv = sep ? ctx->xv : nullptr; a.M = M; a.idx = idx;
      a.light[0] = L[0]; a.light[1] = L[1]; a.light[2] = L[2];
      a.g = ctx->g; a.all_keys = ctx->def_keys; a.owned_max = ctx->owned;
      a.out_rgba = rgba; a.out_depth = depth; a.out_primid = ctx->primid;
      a.sc = ctx->sc;
      a.ctl = ctx->ctl;
      if (ctx->g.NB > 1) a.bin_start = ctx->bin_start;
      CK(launch_shade(a, ctx->pdl, s));
    }
  }
  CK(mark(1 + PIKO_STAGE_RESOLVE));
  if (ev) ++ctx->prof_frames;
  CK(record_frame_end(ctx, s, T, !gather));
  ctx->last_T = T;
  return PIKO_OK;
}

// Expand chunk for the next frames: about RX_CHUNK pairs per chunk given the
// last frame's pairs per triangle (a power of two in [256, EX_MAX_TRIS]).
static void adapt_tri_chunk(piko_ctx* ctx) {
  const double T = (double)ctx->last_T, P = (double)ctx->h_ctl->n_pairs;
  if (T <= 0) return;
  // Expected pairs per chunk at most 3/4 of RX_CHUNK: a chunk over RX_CHUNK
  // takes the windowed slow path (several times slower), and because its group
  // aggregate is then published late it stalls the look-back of every later
  // chunk.  Any multiple of RX_THREADS works (tpt = tri_chunk / RX_THREADS).
  const double want = P > 0 ? 0.75 * RX_CHUNK * T / P : (double)EX_MAX_TRIS;
  long long tc = (long long)(want / RX_THREADS) * RX_THREADS;
#ifndef PIKO_NO_WAVE_CHUNKS
  // Frames with few triangles: shrink chunks while every chunk still fits in
  // one wave of resident radix CTAs.  Smaller chunks finish sooner and are
  // less likely to exceed RX_CHUNK where the pairs per triangle vary a lot
  // (c2: near spheres' triangles cover several bins, far ones one).
  const long long slots = rx_slots(ctx);
  const long long per_wave = ((long long)T + slots - 1) / slots;
  tc = std::min<long long>(tc, (per_wave + RX_THREADS - 1) / RX_THREADS * RX_THREADS);
#endif
  ctx->tri_chunk = (int)std::max<long long>(RX_THREADS, std::min<long long>(EX_MAX_TRIS, tc));
}

// Status of one completed frame from its mirror; PIKO_ECAPACITY (and grown
// capacity) on overflow.  The mirror becomes ctx->h_ctl (stats, chunk sizes).
static int eval_frame(piko_ctx* ctx, piko_ctx::Slot& sl) {
  memcpy(ctx->h_ctl, sl.h, offsetof(Control, digit_hist));
  ctx->last_T = sl.T;
  if (ctx->h_ctl->p2p_timeout) {
    CK(cudaMemsetAsync(&ctx->ctl->p2p_timeout, 0, sizeof(unsigned), 0));
    CK(cudaDeviceSynchronize());
    ctx->last_status = PIKO_ENCCL;
    ctx->fail(PIKO_ENCCL, "P2P exchange: a peer flag wait timed out");
    return ctx->last_status;
  }
  if (ctx->pipeline == PIKO_PIPE_BASELINE &&
      ((long long)ctx->h_ctl->n_pairs > ctx->bl_cap || ctx->h_ctl->vx_overflow)) {
    int rc = ensure_frags(ctx, (long long)ctx->h_ctl->n_pairs);
    if (rc == PIKO_OK) rc = ensure_verts(ctx, (long long)ctx->h_ctl->vx_need);
    ctx->last_status = rc != PIKO_OK ? rc : PIKO_ECAPACITY;
    if (rc == PIKO_OK) ctx->fail(PIKO_ECAPACITY, "fragment capacity exceeded (%llu); grown", ctx->h_ctl->n_pairs);
    return ctx->last_status;
  }
  if (ctx->h_ctl->cl_overflow) ctx->cl_off = true;  // next frames: count matrix (the reset clears the flag)
  if (ctx->h_ctl->overflow_tag == ctx->h_ctl->frame + 1 || ctx->h_ctl->vx_overflow ||
      ctx->h_ctl->peer_overflow == ctx->h_ctl->frame + 1) {
    int rc = ensure_pairs(ctx, ctx->h_ctl->n_pairs);
    if (rc == PIKO_OK) rc = ensure_verts(ctx, (long long)ctx->h_ctl->vx_need);
    ctx->last_status = rc != PIKO_OK ? rc : PIKO_ECAPACITY;
    if (rc == PIKO_OK)
      ctx->fail(PIKO_ECAPACITY, ctx->h_ctl->peer_overflow == ctx->h_ctl->frame + 1
                                    ? "a peer rank's pair capacity was exceeded; its bins are empty"
                                    : "pair capacity exceeded (P=%llu); grown", ctx->h_ctl->n_pairs);
    return ctx->last_status;
  }
  ctx->last_status = PIKO_OK;
  // touched bins per pair over the scatter windows: above 1/4 the rows are
  // dense (coherent meshes: c3 0.02) and the next frames of this size use the
  // radix passes
  if (sl.cm && ctx->h_ctl->n_pairs > 0 && 4 * ctx->h_ctl->cm_touched > ctx->h_ctl->n_pairs)
    ctx->cm_dense_T = sl.T;
  adapt_tri_chunk(ctx);
  return PIKO_OK;
}

// Wait for every frame in flight; the status of the newest one.
static int check_frame(piko_ctx* ctx) {
  const bool had = ctx->ring_n > 0;
  const int rc = poll_frames(ctx, true);
  if (rc != PIKO_OK) return rc;
  return had ? ctx->last_status : ctx->last_status;
}

// A failed CUDA call may leave tickets mid-frame: reset before the next frame.
static int frame_failed(piko_ctx* ctx, int rc) {
  ctx->need_reset = true;
  return rc;
}

static int validate_draw(piko_ctx* ctx, const float* verts, const int32_t* idx, int32_t n_tris,
                         const float* mvp, const float* light, float* rgba, float* depth,
                         float L[3]) {
  if (n_tris < 0) return ctx->fail(PIKO_EINVAL, "n_tris < 0");
  if (!mvp || !light) return ctx->fail(PIKO_EINVAL, "mvp and light must be non-null");
  const bool need_out = !(exchanging(ctx) && ctx->mrank != 0) && !ctx->keys_mode;
  if (need_out && (!rgba || !depth)) return ctx->fail(PIKO_EINVAL, "null output buffer");
  if (n_tris > 0 && (!verts || !idx)) return ctx->fail(PIKO_EINVAL, "null scene buffer");
  if ((reinterpret_cast<uintptr_t>(verts) | reinterpret_cast<uintptr_t>(idx) |
       reinterpret_cast<uintptr_t>(rgba)) & 15u)
    return ctx->fail(PIKO_EINVAL, "verts, idx and out_rgba must be 16-byte aligned");
  for (int k = 0; k < 3; ++k)
    if (!std::isfinite(light[k])) return ctx->fail(PIKO_EINVAL, "light must be finite");
  if (light[0] == 0.0f && light[1] == 0.0f && light[2] == 0.0f)
    return ctx->fail(PIKO_EINVAL, "light must be non-zero");
  for (int k = 0; k < 3; ++k) L[k] = light[k];
  return PIKO_OK;
}

static int draw_impl(piko_ctx* ctx, const float* verts, long long V, const int32_t* idx,
                     int32_t n_tris, const float mvp[16], const float light[3], float* rgba,
                     float* depth, cudaStream_t s, bool force_check, bool force_async,
                     unsigned long long* keys_out = nullptr) {
  float L[3] = {0.0f, 0.0f, 0.0f};
  int rc = validate_draw(ctx, verts, idx, n_tris, mvp, light, rgba, depth, L);
  if (rc != PIKO_OK) return rc;
  CK(cudaSetDevice(ctx->device));
  ctx->prim_base = 0;
  if (ctx->multi == PIKO_MULTI_SORT_LAST && ctx->mnranks > 1) {  // this rank's triangle range
    int64_t t0 = 0, t1 = 0;
    piko_triangle_range(n_tris, ctx->mrank, ctx->mnranks, &t0, &t1);
    idx += 3 * t0;
    n_tris = (int32_t)(t1 - t0);
    ctx->prim_base = t0;
  }
  // statuses of earlier asynchronous frames that have finished (never waits;
  // an overflowed one has grown the capacity before this frame is enqueued)
  if (ctx->pending && (rc = poll_frames(ctx, false)) != PIKO_OK) return rc;
  if (ctx->sticky == PIKO_ECUDA) { ctx->sticky = PIKO_OK; return PIKO_ECUDA; }
  Mat4 M;
  memcpy(M.m, mvp, sizeof M.m);
  if ((rc = ensure_tris(ctx, n_tris)) != PIKO_OK) return rc;
  // without a vertex count the device derives max(idx)+1; start at 3 n_tris
  // (every corner distinct) and grow on a reported vertex overflow
  if (separate_vs(ctx, V, n_tris) && (rc = ensure_verts(ctx, V >= 0 ? V : 3ll * n_tris)) != PIKO_OK) return rc;
  if ((rc = ensure_pairs(ctx, std::max<unsigned long long>(ctx->pair_cap, 2ull * n_tris + 4096))) != PIKO_OK)
    return rc;
  if ((rc = ensure_cov(ctx)) != PIKO_OK) return rc;
  for (int attempt = 0; attempt < 3; ++attempt) {
    if ((rc = enqueue_frame(ctx, verts, V, idx, n_tris, M, L, rgba, depth, s, keys_out)) != PIKO_OK)
      return frame_failed(ctx, rc);
    if ((ctx->sync_mode == PIKO_SYNC_ASYNC || force_async) && !force_check) {
      // enqueued; report (once) an error of an earlier frame
      const int st = ctx->sticky;
      ctx->sticky = PIKO_OK;
      return st;
    }
    rc = check_frame(ctx);
    ctx->sticky = PIKO_OK;  // checked: this frame's status is the answer
    if (rc == PIKO_ECUDA) return frame_failed(ctx, rc);
    if (rc != PIKO_ECAPACITY) return rc;
    // multi-rank: every rank must re-issue together; a capacity miss is
    // reported instead of re-issued so ranks cannot diverge.
    if (exchanging(ctx)) return rc;
  }
  return rc;
}

extern "C" int piko_draw(piko_ctx* ctx, const float* verts, const int32_t* idx, int32_t n_tris,
                         const float mvp[16], const float light[3], float* out_rgba,
                         float* out_depth, void* stream) {
  if (!ctx) return PIKO_EINVAL;
  return draw_impl(ctx, verts, -1, idx, n_tris, mvp, light, out_rgba, out_depth,
                   static_cast<cudaStream_t>(stream), false, false);
}

extern "C" int piko_draw_indexed(piko_ctx* ctx, const float* verts, int64_t n_verts,
                                 const int32_t* idx, int32_t n_tris, const float mvp[16],
                                 const float light[3], float* out_rgba, float* out_depth,
                                 void* stream) {
  if (!ctx) return PIKO_EINVAL;
  if (n_verts < 0 || (n_tris > 0 && n_verts < 1)) return ctx->fail(PIKO_EINVAL, "bad n_verts");
  return draw_impl(ctx, verts, n_verts, idx, n_tris, mvp, light, out_rgba, out_depth,
                   static_cast<cudaStream_t>(stream), false, false);
}

extern "C" int piko_draw_host(piko_ctx* ctx, const float* h_verts, int64_t n_verts,
                              const int32_t* h_idx, int32_t n_tris, const float mvp[16],
                              const float light[3], float* h_rgba, float* h_depth, void* stream) {
  if (!ctx) return PIKO_EINVAL;
  if (n_verts < 0 || n_tris < 0) return ctx->fail(PIKO_EINVAL, "negative size");
  if (n_tris > 0 && (!h_verts || !h_idx)) return ctx->fail(PIKO_EINVAL, "null host scene buffer");
  if (!h_rgba || !h_depth) return ctx->fail(PIKO_EINVAL, "null host output buffer");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(ctx->device));
  const size_t npx = (size_t)ctx->g.W * ctx->g.H;
  if (n_verts > ctx->d_verts_cap) {
    if (ctx->d_verts) cudaFree(ctx->d_verts);
    ctx->d_verts = nullptr;
    CK(cudaMalloc(&ctx->d_verts, sizeof(float) * 8 * std::max<int64_t>(n_verts, 1)));
    ctx->d_verts_cap = n_verts;
  }
  if (n_tris > ctx->d_idx_cap) {
    if (ctx->d_idx) cudaFree(ctx->d_idx);
    ctx->d_idx = nullptr;
    CK(cudaMalloc(&ctx->d_idx, sizeof(int32_t) * 3 * std::max<int32_t>(n_tris, 1)));
    ctx->d_idx_cap = n_tris;
  }
  if (!ctx->d_rgba) {
    CK(cudaMalloc(&ctx->d_rgba, sizeof(float) * 4 * npx));
    CK(cudaMalloc(&ctx->d_depth, sizeof(float) * npx));
  }
  if (n_verts > 0)
    CK(cudaMemcpyAsync(ctx->d_verts, h_verts, sizeof(float) * 8 * n_verts, cudaMemcpyHostToDevice, s));
  if (n_tris > 0)
    CK(cudaMemcpyAsync(ctx->d_idx, h_idx, sizeof(int32_t) * 3 * (size_t)n_tris, cudaMemcpyHostToDevice, s));
  int rc = draw_impl(ctx, ctx->d_verts, n_verts, ctx->d_idx, n_tris, mvp, light, ctx->d_rgba,
                     ctx->d_depth, s, true, false);
  if (rc != PIKO_OK) return rc;
  const bool has_out = !(exchanging(ctx) && ctx->mrank != 0);
  if (has_out) {
    CK(cudaMemcpyAsync(h_rgba, ctx->d_rgba, sizeof(float) * 4 * npx, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(h_depth, ctx->d_depth, sizeof(float) * npx, cudaMemcpyDeviceToHost, s));
  }
  CK(cudaStreamSynchronize(s));
  return PIKO_OK;
}

extern "C" int piko_draw_host_async(piko_ctx* ctx, const float* h_verts, int64_t n_verts,
                                    const int32_t* h_idx, int32_t n_tris, const float mvp[16],
                                    const float light[3], float* h_rgba, float* h_depth, void* stream) {
  if (!ctx) return PIKO_EINVAL;
  if (n_verts < 0 || n_tris < 0) return ctx->fail(PIKO_EINVAL, "negative size");
  if (n_tris > 0 && (!h_verts || !h_idx)) return ctx->fail(PIKO_EINVAL, "null host scene buffer");
  if (!h_rgba || !h_depth) return ctx->fail(PIKO_EINVAL, "null host output buffer");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(ctx->device));
  if (!ctx->cs_in) {
    CK(cudaStreamCreateWithFlags(&ctx->cs_in, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&ctx->cs_out, cudaStreamNonBlocking));
  }
  piko_ctx::HostSlot& h = ctx->hs[ctx->hs_next];
  ctx->hs_next ^= 1;
  const size_t npx = (size_t)ctx->g.W * ctx->g.H;
  if (!h.in_done) {
    CK(cudaEventCreateWithFlags(&h.in_done, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&h.frame_done, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&h.out_done, cudaEventDisableTiming));
    CK(cudaMalloc(&h.rgba, sizeof(float) * 4 * npx));
    CK(cudaMalloc(&h.depth, sizeof(float) * npx));
  }
  if (n_verts > h.vcap || n_tris > h.icap) {  // grow: the slot's last frame must be done with it
    if (h.used) CK(cudaEventSynchronize(h.out_done));
    if (n_verts > h.vcap) {
      if (h.verts) cudaFree(h.verts);
      h.verts = nullptr;
      CK(cudaMalloc(&h.verts, sizeof(float) * 8 * std::max<int64_t>(n_verts, 1)));
      h.vcap = n_verts;
    }
    if (n_tris > h.icap) {
      if (h.idx) cudaFree(h.idx);
      h.idx = nullptr;
      CK(cudaMalloc(&h.idx, sizeof(int32_t) * 3 * std::max<int32_t>(n_tris, 1)));
      h.icap = n_tris;
    }
  }
  // upload (after the slot's previous frame has read its inputs)
  if (h.used) CK(cudaStreamWaitEvent(ctx->cs_in, h.frame_done, 0));
  if (n_verts > 0)
    CK(cudaMemcpyAsync(h.verts, h_verts, sizeof(float) * 8 * n_verts, cudaMemcpyHostToDevice, ctx->cs_in));
  if (n_tris > 0)
    CK(cudaMemcpyAsync(h.idx, h_idx, sizeof(int32_t) * 3 * (size_t)n_tris, cudaMemcpyHostToDevice, ctx->cs_in));
  CK(cudaEventRecord(h.in_done, ctx->cs_in));
  // draw on the caller's stream (enqueue only)
  CK(cudaStreamWaitEvent(s, h.in_done, 0));
  const int rc = draw_impl(ctx, h.verts, n_verts, h.idx, n_tris, mvp, light, h.rgba, h.depth, s, false, true);
  CK(cudaEventRecord(h.frame_done, s));
  // download; the caller's stream then orders after it (its sync covers the frame)
  const bool has_out = !(exchanging(ctx) && ctx->mrank != 0);
  CK(cudaStreamWaitEvent(ctx->cs_out, h.frame_done, 0));
  if (has_out) {
    CK(cudaMemcpyAsync(h_rgba, h.rgba, sizeof(float) * 4 * npx, cudaMemcpyDeviceToHost, ctx->cs_out));
    CK(cudaMemcpyAsync(h_depth, h.depth, sizeof(float) * npx, cudaMemcpyDeviceToHost, ctx->cs_out));
  }
  CK(cudaEventRecord(h.out_done, ctx->cs_out));
  CK(cudaStreamWaitEvent(s, h.out_done, 0));
  h.used = true;
  return rc;
}

// Reyes: Split + Dice on the device into
// context-owned mesh buffers, then the binned pipeline samples the
// micropolygons (the Sample stage: AssignBin + per-bin raster; 32x32 bins in
// the paper) and shades them.  The one host synchronisation is
// the readback of the mesh size between Dice's rate/scan kernel and the mesh
// kernel (the pipeline's grids are sized from the triangle count).
extern "C" int piko_draw_patches(piko_ctx* ctx, const float* patches, int32_t n_patches,
                                 const float mvp[16], const float light[3], float dice_px,
                                 int32_t max_grid, float* out_rgba, float* out_depth, void* stream) {
  if (!ctx) return PIKO_EINVAL;
  if (n_patches < 0 || (n_patches > 0 && !patches) || !mvp || !light)
    return ctx->fail(PIKO_EINVAL, "bad patch arguments");
  if (!(dice_px > 0.0f) || !std::isfinite(dice_px)) return ctx->fail(PIKO_EINVAL, "dice_px must be > 0");
  if (max_grid < 1 || max_grid > 1024 || (max_grid & (max_grid - 1)))
    return ctx->fail(PIKO_EINVAL, "max_grid must be a power of two in [1, 1024]");
  if (reinterpret_cast<uintptr_t>(patches) & 15u) return ctx->fail(PIKO_EINVAL, "patches must be 16-byte aligned");
  if (ctx->pipeline != PIKO_PIPE_BINNED || exchanging(ctx))
    return ctx->fail(PIKO_ESTATE, "piko_draw_patches runs the binned pipeline on one GPU");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(ctx->device));
  if (n_patches > ctx->dice_pcap) {
    if (ctx->dice_rate) cudaFree(ctx->dice_rate);
    if (ctx->dice_base) cudaFree(ctx->dice_base);
    ctx->dice_rate = nullptr; ctx->dice_base = nullptr; ctx->dice_pcap = 0;
    CK(cudaMalloc(&ctx->dice_rate, sizeof(int2) * n_patches));
    CK(cudaMalloc(&ctx->dice_base, sizeof(long long) * 2 * n_patches));
    ctx->dice_pcap = n_patches;
  }
  if (!ctx->dice_total) {
    CK(cudaMalloc(&ctx->dice_total, sizeof(long long) * 2));
    CK(cudaMallocHost(&ctx->h_dice_total, sizeof(long long) * 2));
  }
  DiceArgs d{};
  d.patches = patches; d.n = n_patches; memcpy(d.M.m, mvp, sizeof d.M.m);
  d.W = ctx->g.W; d.H = ctx->g.H; d.dice_px = dice_px; d.max_grid = max_grid;
  d.rate = ctx->dice_rate; d.base = ctx->dice_base; d.total = ctx->dice_total;
  CK(launch_dice_rate(d, s));
  CK(cudaMemcpyAsync(ctx->h_dice_total, ctx->dice_total, sizeof(long long) * 2, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const long long V = ctx->h_dice_total[0], T = ctx->h_dice_total[1];
  if (T > INT32_MAX || V > INT32_MAX) return ctx->fail(PIKO_ECAPACITY, "diced mesh too large (%lld triangles)", T);
  if (V > ctx->dice_vcap) {
    if (ctx->dice_verts) cudaFree(ctx->dice_verts);
    ctx->dice_verts = nullptr; ctx->dice_vcap = 0;
    CK(cudaMalloc(&ctx->dice_verts, sizeof(float) * 8 * std::max<long long>(V, 1)));
    ctx->dice_vcap = std::max<long long>(V, 1);
  }
  if (T > ctx->dice_tcap) {
    if (ctx->dice_idx) cudaFree(ctx->dice_idx);
    ctx->dice_idx = nullptr; ctx->dice_tcap = 0;
    CK(cudaMalloc(&ctx->dice_idx, sizeof(int32_t) * 3 * std::max<long long>(T, 1)));
    ctx->dice_tcap = std::max<long long>(T, 1);
  }
  d.verts = ctx->dice_verts; d.idx = ctx->dice_idx;
  CK(launch_dice(d, s));
  ctx->dice_V = V; ctx->dice_T = T;
  return draw_impl(ctx, ctx->dice_verts, V, ctx->dice_idx, (int32_t)T, mvp, light, out_rgba, out_depth, s, false, false);
}

extern "C" int piko_get_diced(const piko_ctx* ctx, const float** d_verts, int64_t* n_verts,
                              const int32_t** d_idx, int64_t* n_tris) {
  if (!ctx || !d_verts || !n_verts || !d_idx || !n_tris) return PIKO_EINVAL;
  *d_verts = ctx->dice_verts; *n_verts = ctx->dice_V;
  *d_idx = ctx->dice_idx; *n_tris = ctx->dice_T;
  return PIKO_OK;
}

extern "C" int piko_finish(piko_ctx* ctx) {
  if (!ctx) return PIKO_EINVAL;
  int rc = poll_frames(ctx, true);
  if (rc != PIKO_OK) return rc;
  rc = ctx->sticky;  // the first error of any frame since the last report
  ctx->sticky = PIKO_OK;
  return rc;
}

extern "C" int piko_set_sync(piko_ctx* ctx, int mode) {
  if (!ctx) return PIKO_EINVAL;
  if (mode != PIKO_SYNC_CHECKED && mode != PIKO_SYNC_ASYNC) return ctx->fail(PIKO_EINVAL, "bad sync mode");
  ctx->sync_mode = mode;
  return PIKO_OK;
}

extern "C" int piko_get_primid(const piko_ctx* ctx, const int32_t** d_primid) {
  if (!ctx || !d_primid) return PIKO_EINVAL;
  *d_primid = ctx->primid;
  return PIKO_OK;
}

extern "C" int piko_get_bins(const piko_ctx* cctx, const int32_t** d_bin_start,
                             const int32_t** d_bin_prims, int64_t* n_pairs) {
  piko_ctx* ctx = const_cast<piko_ctx*>(cctx);
  if (!ctx || !d_bin_start || !d_bin_prims || !n_pairs) return PIKO_EINVAL;
  if (ctx->pipeline != PIKO_PIPE_BINNED) return ctx->fail(PIKO_ESTATE, "no bin lists outside the binned pipeline");
  int rc = check_frame(ctx);
  if (rc != PIKO_OK) return rc;
  *d_bin_start = ctx->bin_start;
  *d_bin_prims = ctx->prims_out ? ctx->prims_out : ctx->vals[ctx->npass & 1];
  *n_pairs = (int64_t)ctx->h_ctl->n_pairs;
  return PIKO_OK;
}

extern "C" int piko_set_debug(piko_ctx* ctx, unsigned flags) {
  if (!ctx) return PIKO_EINVAL;
  if (flags & ~PIKO_DEBUG_COVERAGE_COUNT) return ctx->fail(PIKO_EINVAL, "unknown debug flag");
  ctx->debug = flags;
  return PIKO_OK;
}

extern "C" int piko_get_coverage(const piko_ctx* ctx, const uint32_t** d_cov) {
  if (!ctx || !d_cov) return PIKO_EINVAL;
  if (!ctx->cov) return PIKO_ESTATE;
  *d_cov = ctx->cov;
  return PIKO_OK;
}

// boundaries are multiples of 4 triangles so idx + 3 t0 keeps idx's 16-byte alignment
extern "C" int piko_triangle_range(int64_t n_tris, int rank, int nranks, int64_t* t0, int64_t* t1) {
  if (n_tris < 0 || nranks < 1 || rank < 0 || rank >= nranks || !t0 || !t1) return PIKO_EINVAL;
  auto cut = [&](int r) -> int64_t { return r >= nranks ? n_tris : (n_tris * r / nranks) & ~int64_t(3); };
  *t0 = cut(rank);
  *t1 = cut(rank + 1);
  return PIKO_OK;
}

extern "C" int piko_set_multi(piko_ctx* ctx, int mode) {
  if (!ctx) return PIKO_EINVAL;
  if (mode != PIKO_MULTI_SORT_FIRST && mode != PIKO_MULTI_SORT_LAST)
    return ctx->fail(PIKO_EINVAL, "unknown multi-GPU mode");
  if (ctx->comm || ctx->p2p_keys) return ctx->fail(PIKO_ESTATE, "ranks attached");
  if (mode == PIKO_MULTI_SORT_LAST && ctx->transport == PIKO_XPORT_P2P)
    return ctx->fail(PIKO_ESTATE, "the P2P transport carries the sort-first tile exchange");
  if (ctx->pending) check_frame(ctx);
  ctx->multi = mode;
  set_ownership(ctx, ctx->mrank, ctx->mnranks);  // re-derive bin ownership
  ctx->need_reset = true;
  return PIKO_OK;
}

// rank 0: exchange buffers + their CUDA IPC handles (keys, sync) into h
static int p2p_export(piko_ctx* ctx, int nranks, void* h) {
  set_ownership(ctx, 0, nranks);
  ctx->transport = PIKO_XPORT_P2P;
  int rc = p2p_alloc(ctx);
  if (rc != PIKO_OK) return rc;
  cudaIpcMemHandle_t* hh = static_cast<cudaIpcMemHandle_t*>(h);
  CK(cudaIpcGetMemHandle(&hh[0], ctx->p2p_keys));
  CK(cudaIpcGetMemHandle(&hh[1], ctx->p2p_sync));
  return PIKO_OK;
}

// rank > 0: map rank 0's exchange buffers
static int p2p_import(piko_ctx* ctx, const void* h, int rank, int nranks) {
  set_ownership(ctx, rank, nranks);
  ctx->transport = PIKO_XPORT_P2P;
  cudaIpcMemHandle_t hh[2];
  memcpy(hh, h, sizeof hh);
  void* pk = nullptr;
  void* ps = nullptr;
  CK(cudaIpcOpenMemHandle(&pk, hh[0], cudaIpcMemLazyEnablePeerAccess));
  CK(cudaIpcOpenMemHandle(&ps, hh[1], cudaIpcMemLazyEnablePeerAccess));
  ctx->p2p_keys = static_cast<unsigned long long*>(pk);
  ctx->p2p_sync = static_cast<unsigned long long*>(ps);
  ctx->p2p_ipc = true;
  return PIKO_OK;
}

static int p2p_check(piko_ctx* ctx, int rank, int nranks) {
  if (nranks < 2 || rank < 0 || rank >= nranks) return ctx->fail(PIKO_EINVAL, "bad rank/nranks");
  if (ctx->comm || ctx->p2p_keys) return ctx->fail(PIKO_ESTATE, "ranks already attached");
  if (ctx->multi != PIKO_MULTI_SORT_FIRST || ctx->pipeline != PIKO_PIPE_BINNED)
    return ctx->fail(PIKO_ESTATE, "P2P peers need sort-first and the binned pipeline");
  CK(cudaSetDevice(ctx->device));
  return PIKO_OK;
}

extern "C" int piko_p2p_export(piko_ctx* ctx, int nranks, void* out_handles) {
  if (!ctx || !out_handles) return PIKO_EINVAL;
  int rc = p2p_check(ctx, 0, nranks);
  return rc != PIKO_OK ? rc : p2p_export(ctx, nranks, out_handles);
}

extern "C" int piko_p2p_import(piko_ctx* ctx, const void* handles, int rank, int nranks) {
  if (!ctx || !handles) return PIKO_EINVAL;
  if (rank == 0) return ctx->fail(PIKO_EINVAL, "rank 0 exports");
  int rc = p2p_check(ctx, rank, nranks);
  return rc != PIKO_OK ? rc : p2p_import(ctx, handles, rank, nranks);
}

extern "C" int piko_set_transport(piko_ctx* ctx, int transport) {
  if (!ctx) return PIKO_EINVAL;
  if (transport != PIKO_XPORT_NCCL && transport != PIKO_XPORT_P2P)
    return ctx->fail(PIKO_EINVAL, "unknown transport");
  if (ctx->comm || ctx->p2p_keys) return ctx->fail(PIKO_ESTATE, "ranks already attached");
  if (transport == PIKO_XPORT_P2P && ctx->multi != PIKO_MULTI_SORT_FIRST)
    return ctx->fail(PIKO_ESTATE, "the P2P transport carries the sort-first tile exchange");
  ctx->transport = transport;
  return PIKO_OK;
}

extern "C" int piko_attach_local_peers(piko_ctx* ctx, piko_ctx* root, int rank, int nranks) {
  if (!ctx || !root) return PIKO_EINVAL;
  if (nranks < 2 || rank < 0 || rank >= nranks) return ctx->fail(PIKO_EINVAL, "bad rank/nranks");
  if ((rank == 0) != (root == ctx)) return ctx->fail(PIKO_EINVAL, "rank 0 is the root context");
  if (ctx->comm || ctx->p2p_keys) return ctx->fail(PIKO_ESTATE, "ranks already attached");
  if (ctx->multi != PIKO_MULTI_SORT_FIRST || ctx->pipeline != PIKO_PIPE_BINNED)
    return ctx->fail(PIKO_ESTATE, "P2P peers need sort-first and the binned pipeline");
  if (root->device != ctx->device || root->g.W != ctx->g.W || root->g.H != ctx->g.H ||
      root->bw != ctx->bw || root->bh != ctx->bh)
    return ctx->fail(PIKO_EINVAL, "root context differs in device, screen or bins");
  if (rank != 0 && (!root->p2p_keys || root->mnranks != nranks))
    return ctx->fail(PIKO_ESTATE, "attach the root (rank 0) first");
  CK(cudaSetDevice(ctx->device));
  set_ownership(ctx, rank, nranks);
  ctx->virt = true;
  ctx->transport = PIKO_XPORT_P2P;
  if (rank == 0) return p2p_alloc(ctx);
  ctx->p2p_keys = root->p2p_keys;
  ctx->p2p_sync = root->p2p_sync;
  return PIKO_OK;
}

extern "C" int piko_set_partition(piko_ctx* ctx, int rank, int nranks) {
  if (!ctx) return PIKO_EINVAL;
  if (ctx->comm || ctx->p2p_keys) return ctx->fail(PIKO_ESTATE, "ranks attached");
  if (nranks < 1 || rank < 0 || rank >= nranks) return ctx->fail(PIKO_EINVAL, "bad rank/nranks");
  if (nranks > 1 && ctx->pipeline != PIKO_PIPE_BINNED)
    return ctx->fail(PIKO_ESTATE, "partitions need the binned pipeline");
  set_ownership(ctx, rank, nranks);
  ctx->virt = nranks > 1;
  return PIKO_OK;
}

extern "C" int piko_attach_comm(piko_ctx* ctx, const void* uid, int rank, int nranks) {
  if (!ctx || !uid) return PIKO_EINVAL;
  if (nranks < 1 || rank < 0 || rank >= nranks) return ctx->fail(PIKO_EINVAL, "bad rank/nranks");
  if (ctx->comm) return ctx->fail(PIKO_ESTATE, "communicator already attached");
  std::string e;
  if (!g_nccl.load(e)) return ctx->fail(PIKO_ENCCL, "%s", e.c_str());
  CK(cudaSetDevice(ctx->device));
  ncclUniqueId id;
  memcpy(&id, uid, sizeof id);
  const int rc = g_nccl.CommInitRank(&ctx->comm, nranks, id, rank);
  if (rc != 0) { ctx->comm = nullptr; return ctx->fail(PIKO_ENCCL, "ncclCommInitRank: %s", g_nccl.GetErrorString(rc)); }
  set_ownership(ctx, rank, nranks);
  if (ctx->transport == PIKO_XPORT_P2P && nranks > 1) {
    // rank 0 allocates the exchange buffers and broadcasts their CUDA IPC
    // handles over the new communicator; the other ranks map them (NVLink P2P)
    unsigned char h[PIKO_P2P_HANDLE_BYTES];
    memset(h, 0, sizeof h);
    if (rank == 0) {
      const int rc0 = p2p_export(ctx, nranks, h);
      if (rc0 != PIKO_OK) return rc0;
    }
    void* d = nullptr;
    CK(cudaMalloc(&d, sizeof h));
    CK(cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice));
    const int rb = g_nccl.Broadcast(d, d, sizeof h, ncclUint8_, 0, ctx->comm, nullptr);
    if (rb != 0) { cudaFree(d); return ctx->fail(PIKO_ENCCL, "ncclBroadcast: %s", g_nccl.GetErrorString(rb)); }
    CK(cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost));  // (synchronises the broadcast)
    CK(cudaFree(d));
    return rank == 0 ? PIKO_OK : p2p_import(ctx, h, rank, nranks);
  }
  // keys of the owned bins + one status word (1: no overflow) that travels
  // with them, so rank 0 learns of a peer's capacity miss
  const size_t words = (size_t)ctx->bw * ctx->bh * std::max(ctx->owned_max, 1) + 1;
  CK(cudaMalloc(&ctx->tile_keys, sizeof(unsigned long long) * words));
  // rank 0's receive buffer: every rank's tiles (sort-first), or one reduced image (sort-last)
  const size_t slots = ctx->multi == PIKO_MULTI_SORT_LAST ? 1 : (size_t)nranks;
  if (rank == 0) CK(cudaMalloc(&ctx->all_keys, sizeof(unsigned long long) * words * slots));
  return PIKO_OK;
}

extern "C" int piko_get_stats(const piko_ctx* cctx, piko_stats* out) {
  piko_ctx* ctx = const_cast<piko_ctx*>(cctx);
  if (!ctx || !out) return PIKO_EINVAL;
  int rc = check_frame(ctx);
  if (rc == PIKO_ECUDA) return rc;
  out->n_tris = ctx->last_T;
  out->n_live = (int64_t)ctx->h_ctl->n_live[ctx->h_ctl->frame & 1];
  out->n_pairs = (int64_t)ctx->h_ctl->n_pairs;
  out->n_bins = ctx->g.NB;
  out->owned_bins = ctx->owned;
  out->pair_capacity = (int64_t)ctx->pair_cap;
  out->radix_passes = ctx->npass;
  out->kernels_per_frame = ctx->last_kernels;
  out->assign_mode = ctx->last_cl ? 2 : ctx->last_cm ? 1 : 0;
  out->reserved = 0;
  out->cm_rows = ctx->last_cl ? ctx->last_cl_nch : ctx->last_cm ? ctx->last_cm_rows : 0;
  return PIKO_OK;
}

extern "C" int piko_nccl_unique_id(void* out) {
  if (!out) return PIKO_EINVAL;
  std::string e;
  if (!g_nccl.load(e)) { g_create_error = e; return PIKO_ENCCL; }
  ncclUniqueId id;
  if (g_nccl.GetUniqueId(&id) != 0) return PIKO_ENCCL;
  memcpy(out, &id, sizeof id);
  return PIKO_OK;
}

extern "C" int piko_set_profiling(piko_ctx* ctx, int on) {
  if (!ctx) return PIKO_EINVAL;
  if (ctx->pending) check_frame(ctx);
  ctx->prof = on != 0;
  ctx->prof_frames = 0;
  return PIKO_OK;
}

extern "C" int piko_get_profile(piko_ctx* ctx, double ms[PIKO_NUM_STAGES], int64_t* frames) {
  if (!ctx || !ms || !frames) return PIKO_EINVAL;
  for (int k = 0; k < PIKO_NUM_STAGES; ++k) ms[k] = 0.0;
  for (long long f = 0; f < ctx->prof_frames; ++f) {
    cudaEvent_t* e = &ctx->ev_pool[(size_t)f * (PIKO_NUM_STAGES + 1)];
    CK(cudaEventSynchronize(e[PIKO_NUM_STAGES]));
    for (int k = 0; k < PIKO_NUM_STAGES; ++k) {
      float t = 0.0f;
      CK(cudaEventElapsedTime(&t, e[k], e[k + 1]));
      ms[k] += t;
    }
  }
  *frames = ctx->prof_frames;
  return PIKO_OK;
}

extern "C" int64_t piko_tile_keys_count(const piko_ctx* ctx) {
  if (!ctx) return PIKO_EINVAL;
  return (int64_t)ctx->owned_max * ctx->bw * ctx->bh;
}

extern "C" int piko_draw_tile_keys(piko_ctx* ctx, const float* verts, int64_t n_verts,
                                   const int32_t* idx, int32_t n_tris, const float mvp[16],
                                   const float light[3], uint64_t* d_tile_keys, void* stream) {
  if (!ctx) return PIKO_EINVAL;
  if (!d_tile_keys) return ctx->fail(PIKO_EINVAL, "null tile-key buffer");
  if (n_verts < 0 || (n_tris > 0 && n_verts < 1)) return ctx->fail(PIKO_EINVAL, "bad n_verts");
  ctx->keys_mode = true;
  const int rc = draw_impl(ctx, verts, n_verts, idx, n_tris, mvp, light, nullptr, nullptr,
                           static_cast<cudaStream_t>(stream), false, false,
                           reinterpret_cast<unsigned long long*>(d_tile_keys));
  ctx->keys_mode = false;
  return rc;
}

extern "C" int piko_resolve_keys(piko_ctx* ctx, const float* verts, int64_t n_verts,
                                 const int32_t* idx, int32_t n_tris, const float mvp[16],
                                 const float light[3], int nranks, const uint64_t* d_all_keys,
                                 float* out_rgba, float* out_depth, void* stream) {
  if (!ctx) return PIKO_EINVAL;
  if (!d_all_keys || !out_rgba || !out_depth || !mvp || !light)
    return ctx->fail(PIKO_EINVAL, "null argument");
  if (nranks < 1 || n_verts < 0 || n_tris < 0) return ctx->fail(PIKO_EINVAL, "bad size");
  float L[3] = {0.0f, 0.0f, 0.0f};
  int rc = validate_draw(ctx, verts, idx, n_tris, mvp, light, out_rgba, out_depth, L);
  if (rc != PIKO_OK) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  CK(cudaSetDevice(ctx->device));
  Mat4 M;
  memcpy(M.m, mvp, sizeof M.m);
  ResolveArgs a{};  // shade re-transforms the winning triangles' corners (no vertex stage)
  a.verts = verts; a.xv = nullptr; a.M = M; a.idx = idx;
  a.light[0] = L[0]; a.light[1] = L[1]; a.light[2] = L[2];
  a.g = ctx->g; a.g.nranks = nranks; a.g.rank = 0;
  a.all_keys = reinterpret_cast<const unsigned long long*>(d_all_keys);
  a.owned_max = (ctx->g.NB + nranks - 1) / nranks;
  a.out_rgba = out_rgba; a.out_depth = out_depth; a.out_primid = ctx->primid;
  CK(launch_resolve(a, false, s));
  return PIKO_OK;
}

extern "C" int64_t piko_owned_bins(int width, int height, int bin_w, int bin_h, int rank,
                                   int nranks, int32_t* out_bins, int64_t cap) {
  if (width < 1 || height < 1 || !pow2_in(bin_w, 8, 64) || !pow2_in(bin_h, 8, 64) || nranks < 1 ||
      rank < 0 || rank >= nranks || cap < 0)
    return PIKO_EINVAL;
  const int64_t NB = (int64_t)((width + bin_w - 1) / bin_w) * ((height + bin_h - 1) / bin_h);
  int64_t n = 0;
  for (int64_t b = rank; b < NB; b += nranks, ++n)
    if (out_bins && n < cap) out_bins[n] = (int32_t)b;
  return n;
}

extern "C" int piko_set_shader_cost(piko_ctx* ctx, int iters, int forward) {
  if (!ctx) return PIKO_EINVAL;
  if (iters < 0 || iters > PIKO_MAX_SHADER_ITERS || (forward != 0 && forward != 1))
    return ctx->fail(PIKO_EINVAL, "shader cost: 0 <= iters <= PIKO_MAX_SHADER_ITERS, forward 0 or 1");
  ctx->sc.iters = iters;
  ctx->sc.forward = forward;
  return PIKO_OK;
}

extern "C" int piko_set_pipeline(piko_ctx* ctx, int pipeline) {
  if (!ctx) return PIKO_EINVAL;
  if (pipeline != PIKO_PIPE_BINNED && pipeline != PIKO_PIPE_FREEPIPE && pipeline != PIKO_PIPE_BASELINE)
    return ctx->fail(PIKO_EINVAL, "unknown pipeline");
  if (pipeline != PIKO_PIPE_BINNED && ctx->mnranks > 1)
    return ctx->fail(PIKO_ESTATE, "FreePipe and Baseline render the whole screen on one GPU");
  if (ctx->pending) check_frame(ctx);
  ctx->pipeline = pipeline;
  ctx->need_reset = true;
  return PIKO_OK;
}
