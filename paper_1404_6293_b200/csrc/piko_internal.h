// piko_internal.h -- structures shared by the kernels (kernels.cu) and the host
// orchestration (piko_api.cu).  Product code only; nothing here is shared with
// the oracle (oracle/piko_oracle.c).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace piko {

// ---- launch geometry -------------------------------------------------------
constexpr int K1_THREADS = 256;                     // vertex+setup+AssignBin CTA
constexpr int K1_TPT = 4;                           // triangles per thread
constexpr int K1_CHUNK = K1_THREADS * K1_TPT;       // triangles per look-back chunk
constexpr int SCAN_THREADS = 256;                   // bin-count scan CTA
constexpr int SCAN_ITEMS = 16;
constexpr int SCAN_CHUNK = SCAN_THREADS * SCAN_ITEMS;
constexpr int RX_THREADS = 256;                     // stable LSD radix pass CTA
constexpr int RX_WARPS = RX_THREADS / 32;
constexpr int RX_ITEMS = 16;
constexpr int RX_CHUNK = RX_THREADS * RX_ITEMS;     // pairs per chunk
constexpr int RX_BITS = 8;
constexpr int RX_RADIX = 1 << RX_BITS;
constexpr int MAX_PASSES = 3;                       // NB <= 2^24 bins

// ---- per-frame device control block (zeroed at frame start) ----------------
struct Control {
  unsigned int ticket_k1;
  unsigned int ticket_scan;
  unsigned int ticket_rx[MAX_PASSES];
  unsigned int overflow;         // K1 saw P > pair capacity
  unsigned long long n_pairs;    // P, written by K1's last chunk
  unsigned long long n_live;     // live (owned) triangles, statistics
  unsigned int digit_hist[MAX_PASSES][RX_RADIX];  // per-pass digit histograms
};

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

struct SetupArgs {
  const float* verts;
  const int32_t* idx;
  long long n_tris;
  Mat4 M;
  Grid g;
  int4* rec;                    // [n_tris][3]
  uint32_t* pair_keys;          // [cap] bin id per pair
  int32_t* pair_vals;           // [cap] primID per pair
  uint32_t* bin_count;          // [NB] pairs per bin (zeroed by k_bin_scan)
  unsigned long long* status;   // [chunks] decoupled look-back
  Control* ctl;
  unsigned long long cap;       // pair capacity
};

struct ScanArgs {
  uint32_t* bin_count;          // [NB] in, zeroed on exit
  int32_t* bin_start;           // [NB+1] out
  unsigned long long* status;   // [chunks]
  Control* ctl;
  int NB;
  int npass;
};

struct RadixArgs {
  const uint32_t* keys_in;
  const int32_t* vals_in;
  uint32_t* keys_out;           // may be null on the last pass
  int32_t* vals_out;
  uint32_t* status;             // [chunks][RX_RADIX]
  Control* ctl;
  int pass;
  int shift;
  unsigned long long cap;
};

struct TileArgs {
  const float* verts;
  const int32_t* idx;
  Mat4 M;
  float light[3];
  Grid g;
  const int4* rec;
  const int32_t* bin_start;
  const int32_t* bin_prims;
  const Control* ctl;
  float* out_rgba;              // may be null (keys-only mode)
  float* out_depth;
  int32_t* out_primid;
  uint32_t* out_cov;            // debug coverage counts or null
  unsigned long long* tile_keys;  // keys-only mode: [owned][bw*bh]
};

struct ResolveArgs {            // rank 0 after the NCCL gather
  const float* verts;
  const int32_t* idx;
  Mat4 M;
  float light[3];
  Grid g;
  const unsigned long long* all_keys;  // [nranks][owned_max][bw*bh]
  int owned_max;
  float* out_rgba;
  float* out_depth;
  int32_t* out_primid;
};

// ---- launchers (kernels.cu) ------------------------------------------------
cudaError_t launch_setup(const SetupArgs& a, int grid, cudaStream_t s);
cudaError_t launch_bin_scan(const ScanArgs& a, int grid, cudaStream_t s);
cudaError_t launch_radix_pass(const RadixArgs& a, int grid, cudaStream_t s);
cudaError_t launch_tile(const TileArgs& a, int bw, int bh, int n_owned_bins, bool cov,
                        bool keys_only, cudaStream_t s);
cudaError_t launch_resolve(const ResolveArgs& a, cudaStream_t s);
// occupancy-derived persistent grid sizes
int max_grid_setup();
int max_grid_scan();
int max_grid_radix();

}  // namespace piko
