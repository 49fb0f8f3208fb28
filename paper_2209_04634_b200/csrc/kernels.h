// kernels.h — host-visible launch interface of the sm_100a kernels.
//
// Parameter structs are passed by value (kernel parameter space); all
// pointers are device pointers.  See DESIGN.md §4 for the data layout.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace evsim_gpu {

constexpr int kWarpsPerBlock = 8;  // chain / emit kernels: 256 threads
constexpr int kMaxLevels = 8;

// ---------------------------------------------------------------- pyramid
struct LevelDims {
  int w, h;
};

// Patch-grid geometry of one pyramid level (flow.cpp:152-171, 220-235).
struct GridGeom {
  int w, h;        // level extent
  int ncx, ncy;    // patch centres per axis
  const int* cx;   // ncx centres  (patch_centers, flow.cpp:97-107)
  const int* cy;   // ncy centres
  const int* ix;   // w   interp_table idx (flow.cpp:111-128)
  const float* wx; // w   interp_table weight
  const int* iy;   // h
  const float* wy; // h
  float* pu;       // ncx*ncy patch-grid flow (u)
  float* pv;       // ncx*ncy patch-grid flow (v)
};

struct DenseLKParams {
  GridGeom g;             // this level
  GridGeom coarse;        // level + 1 (seed source) when has_coarse
  int has_coarse;
  const float* prev;      // level image of prev (w*h fp32)
  const float* curr;      // level image of curr
  int radius;
  int iterations;
};

struct SparseLKParams {
  int levels;
  LevelDims dims[kMaxLevels];
  const float* prev[kMaxLevels];
  const float* curr[kMaxLevels];
  int w0, h0;
  int radius, iterations;
  const uint32_t* points;   // pixel index y*w0+x, scan order
  const int* n_points;      // device count
  int64_t n_points_host;    // used when n_points == nullptr
  float2* disp;
  uint8_t* status;
};

// ---------------------------------------------------------------- chain
enum ProviderKind { kProvNone = 0, kProvDenseGrid = 1, kProvDenseField = 2, kProvSparse = 3 };

// One description of the link chain: chain frame c (c = 0..n_links) is
// frame index start + c*step (0 = prev, 1..N interpolated, N+1 = curr).
struct ChainDesc {
  int start;
  int step;
  int n_links;  // >= 0
};

// Segments = runs of links with equal timestamps (written by scan_kernel,
// read by emit/unpack).  Usually one link per segment.
struct SegTable {
  int* n_segs;       // device scalar
  int* seg_first;    // [max links]
  int* seg_nlinks;   // [max links]
  int64_t* seg_t;    // [max links]
};

struct ChainParams {
  int w, h;
  int wpr;                 // 32-pixel words per row = ceil(w/32)
  int64_t n_words;         // h * wpr
  int words_per_block;
  int n_blocks;
  int n_interp;            // N
  const uint8_t* prev;     // u8 frames
  const uint8_t* curr;
  const uint32_t* qprev;   // quad images (dense provider)
  const uint32_t* qcurr;
  // dense provider, grid form (level-0 patch grid + tables)
  GridGeom g0;
  // dense provider, field form (caller-supplied flow)
  const float* du;
  const float* dv;
  // interpolation constants per chain frame k (0..N+1)
  const double* alpha;     // k/(N+1)
  const double* oma;       // 1.0 - alpha
  const float* fwd;        // (float)alpha
  const float* bwd;        // (float)(1.0 - alpha)
  // sparse provider
  const uint64_t* claims;  // N planes of P keys
  const uint32_t* touched; // ceil(N/32) planes of P bits
  uint64_t* claims_rw;
  uint32_t* touched_rw;
  const uint32_t* points;  // selected pixel indices
  const int* d_direct;     // when non-null: *d_direct == 0 selects `direct` chain
  // chain descriptions
  ChainDesc full;
  ChainDesc direct;
  // event rule
  int log_mode;
  int magnitude;
  int c_pos, c_neg;
  float c_pos_log, c_neg_log;
  const float* lut;        // 256 log LUT (log mode)
  float* ref;              // P log reference state (log mode)
  // outputs
  uint2* masks;            // [link][n_words] (pos, neg)
  uint16_t* mcount;        // magnitude: [link][n_words*32]
  uint32_t* wcount;        // magnitude: [link][n_words]
  uint32_t* counts;        // [link][n_blocks]
};

struct ScanParams {
  int n_blocks;
  const uint32_t* counts;  // [link][n_blocks]
  const int* d_direct;
  ChainDesc full;
  ChainDesc direct;
  int n_interp;            // timestamps: sub_interval_end over (t_prev, t_curr]
  int64_t t_prev, t_curr;
  SegTable seg;
  int64_t* offsets;        // [seg][n_blocks] exclusive, segment-major
  int64_t* seg_out;        // [0] = n_segs, [1..n_segs] seg_t, then n_segs+1 offsets
  int64_t* total;          // device total
  int64_t* host_total;     // host-mapped mirror (may be null)
};

struct EmitParams {
  int w, h, wpr;
  int64_t n_words;
  int words_per_block;
  int n_blocks;
  const int* d_direct;
  ChainDesc full;
  ChainDesc direct;
  SegTable seg;
  int magnitude;
  const uint2* masks;
  const uint16_t* mcount;
  const uint32_t* wcount;
  const int64_t* offsets;
  const int64_t* total;
  int64_t capacity;
  uint32_t* out;
};

// ---------------------------------------------------------------- sparse
struct SelectParams {
  int w, h, wpr;
  int64_t n_words;
  int words_per_block;
  int n_blocks;
  const uint8_t* prev;
  const uint8_t* curr;
  int log_mode;
  int sel;
  float sel_log;
  const float* lut;
  uint32_t* masks;        // [n_words]
  uint32_t* counts;       // [n_blocks]
  int64_t* offsets;       // [n_blocks] scratch
  uint32_t* points;       // out: pixel indices
  int* n_points;          // out: M
};

struct SplatParams {
  int w, h;
  int n_interp;
  const uint32_t* points;
  const int* n_points;
  const float2* disp;
  const uint8_t* status;
  const uint8_t* prev;
  uint64_t* claims;
  uint32_t* touched;
};

// ---------------------------------------------------------------- launches
void launch_to_float(const uint8_t* src, float* dst, int64_t n, cudaStream_t s);
void launch_downsample(const float* src, LevelDims sd, float* dst, LevelDims dd, cudaStream_t s);
void launch_build_quad(const uint8_t* src, uint32_t* dst, int w, int h, cudaStream_t s);
void launch_dense_lk(const DenseLKParams& p, cudaStream_t s);
void launch_densify(const GridGeom& g, float* du, float* dv, cudaStream_t s);
void launch_interp_frames(const ChainParams& p, uint8_t* out, cudaStream_t s);
void launch_chain(const ChainParams& p, int provider, cudaStream_t s);
void launch_scan(const ScanParams& p, cudaStream_t s);
void launch_emit(const EmitParams& p, cudaStream_t s);
void launch_select(const SelectParams& p, cudaStream_t s);
void launch_select_emit(const SelectParams& p, const int64_t* total, cudaStream_t s);
void launch_init_ref(const uint8_t* frame, const float* lut, float* ref, int64_t n, cudaStream_t s);
void launch_sparse_lk(const SparseLKParams& p, int max_points, cudaStream_t s);
void launch_splat(const SplatParams& p, int max_points, cudaStream_t s);
void launch_unpack_events(const uint32_t* packed, const int64_t* seg_out, int64_t n, void* out24,
                          cudaStream_t s);

}  // namespace evsim_gpu
