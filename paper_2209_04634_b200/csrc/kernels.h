// kernels.h — host-visible launch interface of the sm_100a kernels.
//
// Parameter structs are passed by value (kernel parameter space); all
// pointers are device pointers.  See DESIGN.md §4 for the data layout.
//
// Batching: one launch sequence processes F consecutive frame PAIRS of one
// stream.  Frames live in a device ring of R slots; pair i (0..F-1) reads
// prev = slot (r0 + i) % R and curr = slot (r0 + i + 1) % R.  Everything a
// pair owns (patch grids, sparse points/claims, chain masks) is indexed by i.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "evsim_gpu.h"

namespace evsim_gpu {

constexpr int kWarpsPerBlock = 8;  // chain / emit kernels: 256 threads
constexpr int kMaxLevels = 8;
constexpr int kMaxBatch = 1024;    // frames per push_frames call
constexpr int kChainBias = 0x4B000000;  // dense chain values: the fp32 bits of 2^23 + v (an int compare orders them)
constexpr int kMaxParamK = 64;     // chain frames (N + 2) whose constants travel in the kernel parameters

struct LevelDims {
  int w, h;
};

// A per-slot device array: element (slot, i) at base[slot * stride + i].
template <class T>
struct Ring {
  T* base;
  size_t stride;
  __host__ __device__ T* at(int slot) const { return base + (size_t)slot * stride; }
};

// ---------------------------------------------------------------- pyramid
struct PyramidParams {
  int levels;
  LevelDims dims[kMaxLevels];
  Ring<const uint8_t> frames;
  Ring<float> pyr[kMaxLevels];
  Ring<float4> qpyr[kMaxLevels];
  Ring<uint32_t> quad_u8;   // base may be null (no interpolation)
  Ring<float4> tex[kMaxLevels];  // sparse: per pixel (value, gx, gy, 0); base may be null
  Ring<uint32_t> tex8;           // sparse, u8 level 0: packed texels value | (2gx & 511) << 8 | (2gy & 511) << 17
  int u8_level0;            // level 0 not materialised as fp32 (dense: the solver reads the u8 frame / quad)
  int R, slot0;             // frame j of this launch is slot (slot0 + j) % R
};

// Patch-grid geometry of one pyramid level (flow.cpp:152-171, 220-235).
// pu/pv: per-pair patch grids, pair i at pu + i * pair_stride.
struct GridGeom {
  int w, h;        // level extent
  int ncx, ncy;    // patch centres per axis
  const int* cx;   // ncx centres  (patch_centers, flow.cpp:97-107)
  const int* cy;   // ncy centres
  const int* ix;   // w   interp_table idx (flow.cpp:111-128)
  const float* wx; // w   interp_table weight
  const int* iy;   // h
  const float* wy; // h
  float* pu;
  float* pv;
  size_t pair_stride;
};

struct DenseLKParams {
  int jt0, jt1;           // patch rows [jt0, jt1) to solve (row bands; full grid otherwise)
  GridGeom g;             // this level
  GridGeom coarse;        // level + 1 (seed source) when has_coarse
  int has_coarse;
  Ring<const float> prev; // level images
  Ring<const float4> qcurr;
  int u8;                  // level 0 from the u8 frame ring / u8 quad ring instead
  Ring<const uint8_t> prev8;
  Ring<const uint32_t> qcurr8;
  int R, r0;              // pair z: prev slot (r0+z)%R, curr slot (r0+z+1)%R
  int radius;
  int iterations;
};

struct SparseLKParams {
  int levels;
  LevelDims dims[kMaxLevels];
  Ring<const float4> tex[kMaxLevels];    // prev: (value, gx, gy, 0) per pixel
  Ring<const float4> qcurr[kMaxLevels];  // curr: quad images
  int u8_level0;                         // level 0 from the packed u8 texels / u8 quads below
  Ring<const uint32_t> tex8;             // prev, level 0: packed (value, 2gx, 2gy)
  Ring<const uint32_t> qcurr8;           // curr, level 0: u8 quads
  int R, r0;
  int w0, h0;
  int radius, iterations;
  const uint32_t* points;   // pair i at points + i * P (pixel index y*w0+x, scan order)
  const int* n_points;      // [pairs] device counts, or null
  int64_t n_points_host;    // used when n_points == nullptr (single pair)
  float2* disp;             // pair i at + i * P
  uint8_t* status;          // pair i at + i * P
  size_t pair_stride;       // P
};

// ---------------------------------------------------------------- chain
enum ProviderKind { kProvNone = 0, kProvDenseGrid = 1, kProvDenseField = 2, kProvSparse = 3, kProvDiffInterp = 4 };

// Chain frame c (c = 0..n_links) of every pair is frame index start + c*step
// (0 = prev, 1..N interpolated, N+1 = curr).
struct ChainDesc {
  int start;
  int step;
  int n_links;  // >= 0, per pair
};

// Segments = runs of (pair, link) with equal timestamps, over all links of
// the launch (link g = pair * n_links + l).  Built by segments_kernel.
struct SegTable {
  int* n_segs;       // device scalar
  int* seg_first;    // [links]
  int* seg_nlinks;   // [links]
  int64_t* seg_t;    // [links]
};

struct SegParams {
  ChainDesc d;
  int n_pairs;
  int n_interp;
  SegTable seg;
  int64_t ts[kMaxBatch + 1];  // frame timestamps: pair i = (ts[i], ts[i+1]]
};

struct ChainParams {
  int w, h;
  int row0;                // first frame row of the word grid (row bands; 0 = full frame)
  int wpr;                 // 32-pixel words per row = ceil(w/32)
  int64_t n_words;         // h * wpr
  int words_per_block;
  int n_blocks;
  int words_per_warp;      // 32-pixel words a warp evaluates together (the dense chain: 1)
  int n_interp;            // N
  int n_pairs;
  int R, r0;
  Ring<const uint8_t> frames;
  Ring<const uint32_t> quads;  // u8 quad images (dense provider)
  Ring<const float4> quadf;    // dense chain: fp32 lerp quads of the same frames (base null: not used)
  Ring<const uint2> quadh;     // dense chain: bf16 lerp quads (base null: not used)
  // tile-staged dense chain (chain_dense_tile_kernel): per pixel the top pair
  // (a00, a10 - a00) in fp32, staged per (tile, pair) in shared memory; base
  // null: not used.  tile_cap_rows = staging rows per block, tile_min_blocks =
  // resident blocks per SM the launch asks for (3 or 4)
  Ring<const float2> quadt;
  int tile_cap_rows;
  int tile_min_blocks;
  // difference_only device pushes read the caller's frames in place:
  // pair i = (i ? dcurr + (i-1)*P : dprev, dcurr + i*P); null = the ring
  const uint8_t* dcurr;
  const uint8_t* dprev;
  float magic_y;               // dense chain: Y truncation magic 2^23 + m_y (exact integer float)
  uint32_t qshift;             // dense chain: (bits(2^23 + m_y) * w + bits(2^23)) mod 2^32, + w*h <= 2^32
  // dense provider, grid form (level-0 patch grid + tables; per-pair pu/pv)
  GridGeom g0;
  // dense provider, field form (caller-supplied flow, single pair)
  const float* du;
  const float* dv;
  // interpolation constants per chain frame k (0..N+1)
  const double* alpha;     // k/(N+1)
  const double* oma;       // 1.0 - alpha
  const float* fwd;        // (float)alpha
  const float* bwd;        // (float)(1.0 - alpha)
  const float* alpha_f;    // (float)alpha   (fp32 blend estimate)
  const float* oma_f;      // (float)oma
  const float2* nfb;       // (-(float)alpha, (float)(1.0 - alpha))
  const float4* kc;        // (-(float)alpha, (float)(1 - alpha), (float)oma, (float)alpha)
  // the dense chain's copy of kc in the parameter space (constant bank: the
  // per-link loads go through the constant cache, not the L1 data pipe);
  // N + 2 <= kMaxParamK, larger N use the generic chain kernel
  float4 kcp[kMaxParamK];
  const int4* lthr;        // log mode: per reference level r (0..255): biased (hi, lo) thresholds, L[r] bits, 0
  // sparse provider (per pair strides)
  uint32_t* claims;        // [pair][N][P] keys (change << 24 | ~j)
  uint32_t* touched;       // [pair][ceil(N/32)][P] bits
  const uint8_t* svals;    // [pair][N][P] winning splat values (valid where touched)
  const int16_t* dvals;    // difference_interp: [pair][N][P] winning signed differences
  int skip_first;          // difference_interp: pair 0 has no previous difference frame
  const uint32_t* points;  // [pair][P]
  const int* n_points;     // [pair]
  size_t P;
  int skip_empty;          // log mode without endpoints: M == 0 pairs emit nothing
  ChainDesc d;
  // event rule
  int log_mode;
  int magnitude;
  int c_pos, c_neg;
  float c_pos_log, c_neg_log;
  const float* lut;        // 256 log LUT (log mode)
  float* ref;              // P log reference state (log mode)
  // outputs (link g = pair * d.n_links + l)
  uint2* masks;            // [g][n_words] (pos, neg)
  uint16_t* mcount;        // magnitude: [g][n_words*32]
  uint32_t* wcount;        // magnitude: [g][n_words]
  uint32_t* counts;        // [g][n_blocks] events per block
  unsigned int* sched;     // sparse chain: device task counter (zeroed by the launch)
  size_t masks_cap;        // elements of masks / counts (checked build: EVSIM_CHECK)
  size_t counts_cap;
};

struct OffsetParams {
  int n_rows;              // links
  int n_blocks;
  const uint32_t* counts;  // [g][n_blocks]
  int64_t* prefix;         // [g][n_blocks] exclusive
  int64_t* link_total;     // [g]
};

// n / d for n < 2^27 by one wide multiply and a shift (d >= 1): s = 27 +
// ceil(log2 d), m = ceil(2^s / d) < 2^28, and m*d - 2^s < d <= 2^(s-27)
// makes floor(n*m / 2^s) = floor(n / d) exact (Granlund-Montgomery).
struct FastDiv {
  uint32_t m = 1;
  int s = 0;
  __host__ __device__ uint32_t div(uint32_t n) const {
    return (uint32_t)(((unsigned long long)n * m) >> s);
  }
  static FastDiv make(uint32_t d) {
    FastDiv f;
    int l = 0;
    while ((1ull << l) < d) ++l;
    f.s = 27 + l;
    f.m = (uint32_t)(((1ull << f.s) + d - 1) / d);
    return f;
  }
};

struct EmitParams {
  int w, h, wpr;
  FastDiv wdiv;            // / wpr (word index -> row)
  int row0;                // first frame row of the word grid
  int64_t n_words;
  int words_per_block;
  int n_blocks;
  int n_links;             // links of the launch (pairs * per-pair links)
  int seg_lo, seg_hi;      // segments this launch emits: [seg_lo, seg_hi), or all when seg_hi == 0
  SegTable seg;
  const int64_t* prefix;
  const uint32_t* counts;  // [g][n_blocks] events per (link, block)
  const int64_t* link_total;
  int64_t* seg_out;        // [0] = S, [1..S] seg_t, [1+S..1+2S] offsets (S+1); block 0
  int64_t* base;           // device scalar: output offset of this launch's first event;
                           // segbase_kernel advances it by the launch's total
  int magnitude;
  const uint2* masks;
  const uint16_t* mcount;
  const uint32_t* wcount;
  int64_t capacity;
  uint32_t* out;
};

// wire format (wire_kernels.cu)
struct WireParams {
  int n_links;               // links of the launch
  int64_t n_words;
  int words_per_block;       // the chain's block geometry
  int n_blocks;
  int blocks_per_tile;       // chain blocks per wire CTA (<= 256 words)
  const uint2* masks;        // [g][n_words] (pos, neg)
  const int64_t* prefix;     // [g][n_blocks] exclusive event prefix within the link
  const int64_t* link_total; // [g]
  int64_t* link_bit;         // [g] out: first polarity bit of link g (call-wide numbering)
  int64_t* link_count;       // [g] out: events of link g
  int64_t* bit_base;         // device scalar: the call's next free polarity bit (advanced)
  uint32_t* planes;          // [g][n_words] out
  uint32_t* pol;             // the call's polarity words (zeroed at the call start)
};

// ---------------------------------------------------------------- sparse
struct SelectParams {
  int w, h, wpr;
  int64_t n_words;
  int words_per_block;
  int n_blocks;
  int R, r0;
  Ring<const uint8_t> frames;
  int log_mode;
  int sel;
  float sel_log;
  const float* lut;
  int diff_mode;          // difference_interp: active points of d1 = f[r0+z] - f[r0+z-1]
  int c_pos, c_neg;       //   (simulate.cpp:78-87)
  int skip_first;         //   pair 0 has no d1: selects nothing
  uint32_t* masks;        // [pair][n_words]
  uint32_t* counts;       // [pair][n_blocks]
  int64_t* prefix;        // [pair][n_blocks] exclusive prefix of counts
  int64_t* total;         // [pair]
  uint32_t* points;       // [pair][P]
  int* n_points;          // [pair]
  size_t P;
};

struct SplatParams {
  int w, h;
  int n_interp;
  int R, r0;
  Ring<const uint8_t> frames;
  const uint32_t* points;  // [pair][P]
  const int* n_points;     // [pair]
  const float2* disp;      // [pair][P]
  const uint8_t* status;   // [pair][P]
  uint32_t* claims;        // [pair][N][P]
  uint32_t* touched;       // [pair][ceil(N/32)][P]
  uint8_t* svals;          // [pair][N][P]
  int diff_mode;           // difference_interp: signed d1 values, claims by |d1|
  int16_t* dvals;          // [pair][N][P] (difference_interp)
  size_t P;
};

// ---------------------------------------------------------------- launches
void launch_pyramid(const PyramidParams& p, int n_frames, cudaStream_t s);
void launch_build_quad(const uint8_t* src, uint32_t* dst, int w, int h, cudaStream_t s);
void launch_dense_lk(const DenseLKParams& p, int n_pairs, cudaStream_t s);
void launch_densify(const GridGeom& g, float* du, float* dv, cudaStream_t s);
// the dense chain's fp32 / bf16 lerp quads of n_frames ring slots from slot0
// widest frame whose fp32 lerp quads (tap-relative constants a00 - x*dx, dy -
// x*dxy) are exact integers below 2^24: 255 + 510 * (w - 1) < 2^24
constexpr int kLerpQuadMaxW = 32768;
void launch_lerp_quads(Ring<const uint8_t> frames, Ring<float4> out, int w, int h, int R, int slot0, int n_frames,
                       cudaStream_t s);
void launch_lerp_quads_f2(Ring<const uint8_t> frames, Ring<float2> out, int w, int h, int R, int slot0, int n_frames,
                          cudaStream_t s);
void launch_lerp_quads_bf16(Ring<const uint8_t> frames, Ring<uint2> out, int w, int h, int R, int slot0, int n_frames,
                            cudaStream_t s);
void launch_interp_frames(const ChainParams& p, uint8_t* out, cudaStream_t s);
void launch_segments(const SegParams& p, cudaStream_t s);
// per-(function, device) MaxDynamicSharedMemorySize, thread-safe; throws
// std::runtime_error if the driver refuses
void set_max_dynamic_smem(const void* func, int bytes);
void launch_chain(const ChainParams& p, int provider, cudaStream_t s);
void launch_offsets(const OffsetParams& p, cudaStream_t s);
void launch_emit(const EmitParams& p, int64_t* segbase, cudaStream_t s);
// every link of [g0, g1) its own segment, single mode: segbase + the
// tile-staged emit; false (nothing launched) when it does not apply
bool launch_emit_single(const EmitParams& p, int64_t* segbase, int g0, int g1, cudaStream_t s);
void launch_segbase(const EmitParams& p, int64_t* segbase, cudaStream_t s);
void launch_wire(const WireParams& p, cudaStream_t s);
// segment s of a packed stream ([off[s], off[s+1])) to dst + dst_off[s] (dst may be peer memory)
void launch_place(const uint32_t* src, const int64_t* off, const int64_t* dst_off, int n_segs, int64_t max_len,
                  uint32_t* dst, cudaStream_t s);
void launch_select(const SelectParams& p, int n_pairs, cudaStream_t s);
void launch_init_ref(const uint8_t* frame, const float* lut, float* ref, int64_t n, cudaStream_t s);
// mags[slot] = min(255, |f[slot] - f[slot-1]|) for n consecutive ring slots from slot0
void launch_mags(Ring<const uint8_t> frames, Ring<uint8_t> mags, int R, int slot0, int n, size_t P, cudaStream_t s);
void launch_sparse_lk(const SparseLKParams& p, int max_points, int n_pairs, cudaStream_t s);
void launch_splat(const SplatParams& p, int max_items, int n_pairs, cudaStream_t s);
void launch_unpack_events(const uint32_t* packed, const int64_t* seg_out, int64_t n, void* out24,
                          cudaStream_t s);

// io_kernels.cu — frame ingestion, .evs records, metrics
void launch_luma(const uint8_t* rgb, uint8_t* out, int64_t n, cudaStream_t s);
void launch_resize(const uint8_t* src, int w, int h, uint8_t* dst, int tw, int th, int n_frames, cudaStream_t s);
void launch_evs_records(const uint32_t* packed, const int64_t* seg_out, int64_t n, uint8_t* out, cudaStream_t s);
// core.hpp free functions (core.cpp:5-46): difference_frame and threshold_events
void launch_difference(const uint8_t* prev, const uint8_t* curr, int16_t* out, int64_t n, cudaStream_t s);
int64_t threshold_tiles(int64_t n);
void launch_threshold_count(const int16_t* v, int64_t n, int c_pos, int c_neg, int mag, int64_t* tile_total,
                            cudaStream_t s);
void launch_threshold_emit(const int16_t* v, int64_t n, int w, int c_pos, int c_neg, int mag, int64_t t,
                           const int64_t* tile_off, evsim_event* out, cudaStream_t s);
void launch_event_counts(const evsim_event* ev, int64_t n, int w, uint32_t* counts, cudaStream_t s);
void launch_accumulate(const evsim_event* ev, int64_t n, int w, int64_t t0, int64_t t1, uint32_t* bits,
                       uint8_t* classes, int64_t P, cudaStream_t s);

}  // namespace evsim_gpu
