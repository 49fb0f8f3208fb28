// event_kernels.cu — interpolation + difference/threshold chain, ordered
// compaction, sparse selection and splat (sm_100a).
//
// Replaces src/simulate.cpp:91-201 and src/core.cpp:5-46 of the reference
// (/root/reference/proj).  Layout: every link of every frame
// pair of a launch is evaluated per pixel in one pass; a warp covers 32
// consecutive pixels of one row (a "word") and publishes each link's
// positive / negative crossings as two 32-bit ballots, plus per-(link, block)
// event counts.  offsets/segbase turn the counts into output positions and
// the emit kernel writes every event exactly once, contiguously, in the
// reference's order (t, y, x, p).
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <mutex>
#include <set>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>

#include "evsim_device.cuh"
#include "kernels.h"

namespace evsim_gpu {

namespace {

__device__ __forceinline__ int64_t sub_interval_end(int64_t t0, int64_t t1, int k, int n_steps) {
  // include/evsim/simulate.hpp:15-19
  const int64_t dt = t1 - t0;
  const int64_t num = (int64_t)k * dt;
  return t0 + (num + n_steps - 1) / n_steps;
}

// Block-wide exclusive scan of one value per thread (blockDim.x <= 1024).
template <class T>
__device__ __forceinline__ T block_exclusive_scan(T v, T* s_warp, T& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    T w = lane < nw ? s_warp[lane] : T(0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T y = __shfl_up_sync(kFull, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) s_warp[lane] = w;
  }
  __syncthreads();
  total = s_warp[nw - 1];
  const T before = warp ? s_warp[warp - 1] : T(0);
  __syncthreads();
  return before + x - v;
}

// ------------------------------------------------------------ value providers
// value(k) = intensity of chain frame k of one pair at this pixel: k = 0
// prev, k = N+1 curr, 1..N the interpolated / splatted frame.

struct PixelCtx {
  bool valid;  // false for padding lanes (beyond the row) and duplicate words
  int x, y;
  size_t pix;
  float xf, yf;
};

// Everything one frame pair of the launch reads.
struct PairCtx {
  const uint8_t* prev;
  const uint8_t* curr;
  const uint32_t* qprev;
  const uint32_t* qcurr;
  const float* pu;
  const float* pv;
  uint32_t* claims;
  uint32_t* touched;
  const uint32_t* points;
  bool skip;  // emits nothing (log mode, no endpoints, empty sparse selection)
};

__device__ __forceinline__ PairCtx pair_ctx(const ChainParams& p, int i) {
  PairCtx c;
  const int sp = (p.r0 + i) % p.R, sc = (p.r0 + i + 1) % p.R;
  c.prev = p.frames.at(sp);
  c.curr = p.frames.at(sc);
  c.qprev = p.quads.base ? p.quads.at(sp) : nullptr;
  c.qcurr = p.quads.base ? p.quads.at(sc) : nullptr;
  c.pu = p.g0.pu ? p.g0.pu + (size_t)i * p.g0.pair_stride : nullptr;
  c.pv = p.g0.pv ? p.g0.pv + (size_t)i * p.g0.pair_stride : nullptr;
  const int nw = (p.n_interp + 31) >> 5;
  c.claims = p.claims ? p.claims + (size_t)i * p.n_interp * p.P : nullptr;
  c.touched = p.touched ? p.touched + (size_t)i * nw * p.P : nullptr;
  c.points = p.points ? p.points + (size_t)i * p.P : nullptr;
  c.skip = p.skip_empty && p.n_points && p.n_points[i] == 0;
  return c;
}

// Dense: flow-based two-sided interpolation, interpolate_frames
// (simulate.cpp:91-121), with the flow either densified from the pair's
// level-0 patch grid (flow.cpp:224-245) or read from a caller-supplied field.
template <bool kField>
struct DenseProvider {
  float u, v;
  __device__ __forceinline__ void init(const ChainParams& p, const PairCtx& pc, const PixelCtx& c);
  __device__ __forceinline__ int interp(const ChainParams& p, const PairCtx& pc, const PixelCtx& c, int k) const {
    const float fwd = __ldg(p.fwd + k);
    const float bwd = __ldg(p.bwd + k);
    const float xp = fsub(c.xf, fmul(fwd, u)), yp = fsub(c.yf, fmul(fwd, v));
    const float xc = fadd(c.xf, fmul(bwd, u)), yc = fadd(c.yf, fmul(bwd, v));
    if constexpr (kField) {
      // caller-supplied flow may hold NaN: the reference's exact clamp path
      const float fp = sample_quad(pc.qprev, p.w, p.h, xp, yp);
      const float fc = sample_quad(pc.qcurr, p.w, p.h, xc, yc);
      const double blend = dadd(dmul(__ldg(p.oma + k), (double)fp), dmul(__ldg(p.alpha + k), (double)fc));
      return lround_pos(blend);
    } else {
      // our densified flow is finite: both samples as fp32x2 pairs,
      // conversion-free; (xf - fwd*u, xf + bwd*u) = xf + (-fwd, bwd)*u exactly
      (void)xp, (void)yp, (void)xc, (void)yc;
      const float2 nb = __ldg(p.nfb + k);
      const f32x2 NB = pk2(nb.x, nb.y);
      const f32x2 S = sample_quad_pair(pc.qprev, pc.qcurr, p.w, p.h, affine2(c.xf, NB, u), affine2(c.yf, NB, v));
      const float fp = lo2(S), fc = hi2(S);
      // The reference rounds s = RN64(RN64(oma*fp) + RN64(alpha*fc))
      // (simulate.cpp:114).  An fp32 estimate e of it satisfies
      // |e - s| <= 2^-24*255 + 2^-23*255 + 2^-24*256 + 3*2^-53*256 < 6.2e-5,
      // so lround(s) = trunc(e) + (frac(e) > 0.5) whenever |frac(e) - 0.5| >
      // 1e-4; only inside that window is the double expression evaluated.
      const float e = __fmaf_rn(__ldg(p.oma_f + k), fp, __fmul_rn(__ldg(p.alpha_f + k), fc));
      int n;
      const float fr = fsub(e, trunc_magic(e, n));
      if (fabsf(fsub(fr, 0.5f)) > 1e-4f) return n + (fr > 0.5f ? 1 : 0);
      const double blend = dadd(dmul(__ldg(p.oma + k), (double)fp), dmul(__ldg(p.alpha + k), (double)fc));
      return lround_pos_fast(blend);
    }
  }
  __device__ __forceinline__ void finish(const ChainParams&, const PairCtx&, const PixelCtx&) const {}
};

template <>
__device__ __forceinline__ void DenseProvider<false>::init(const ChainParams& p, const PairCtx& pc,
                                                          const PixelCtx& c) {
  const GridGeom& g = p.g0;
  const int j = __ldg(g.iy + c.y);
  const float fy = __ldg(g.wy + c.y);
  const int i = __ldg(g.ix + c.x);
  const float fx = __ldg(g.wx + c.x);
  const int i0 = min(i, g.ncx - 1), i1 = min(i + 1, g.ncx - 1);
  const int j0 = min(j, g.ncy - 1), j1 = min(j + 1, g.ncy - 1);
  const size_t r0 = (size_t)j0 * g.ncx, r1 = (size_t)j1 * g.ncx;
  const float u_top = lerp_ref(__ldg(pc.pu + r0 + i0), __ldg(pc.pu + r0 + i1), fx);
  const float u_bot = lerp_ref(__ldg(pc.pu + r1 + i0), __ldg(pc.pu + r1 + i1), fx);
  const float v_top = lerp_ref(__ldg(pc.pv + r0 + i0), __ldg(pc.pv + r0 + i1), fx);
  const float v_bot = lerp_ref(__ldg(pc.pv + r1 + i0), __ldg(pc.pv + r1 + i1), fx);
  u = lerp_ref(u_top, u_bot, fy);
  v = lerp_ref(v_top, v_bot, fy);
}
template <>
__device__ __forceinline__ void DenseProvider<true>::init(const ChainParams& p, const PairCtx&, const PixelCtx& c) {
  u = __ldg(p.du + c.pix);
  v = __ldg(p.dv + c.pix);
}

// No intermediate frames: chains over prev/curr only (difference_only, N = 0).
struct NoneProvider {
  __device__ __forceinline__ void init(const ChainParams&, const PairCtx&, const PixelCtx&) {}
  __device__ __forceinline__ int interp(const ChainParams&, const PairCtx& pc, const PixelCtx& c, int) const {
    return pc.prev[c.pix];
  }
  __device__ __forceinline__ void finish(const ChainParams&, const PairCtx&, const PixelCtx&) const {}
};

template <class Prov>
__device__ __forceinline__ int frame_value(const ChainParams& p, const Prov& prov, const PairCtx& pc,
                                           const PixelCtx& c, int k) {
  if (k == 0) return pc.prev[c.pix];
  if (k == p.n_interp + 1) return pc.curr[c.pix];
  return prov.interp(p, pc, c, k);
}

// Position of the (r+1)-th set bit of m (r >= 0, r < popc(m)): a branch-free
// binary search on popcounts.
__device__ __forceinline__ int nth_set_bit(uint32_t m, int r) {
  int pos = 0;
  int c = __popc(m & 0xFFFFu);
  if (r >= c) r -= c, m >>= 16, pos += 16;
  c = __popc(m & 0xFFu);
  if (r >= c) r -= c, m >>= 8, pos += 8;
  c = __popc(m & 0xFu);
  if (r >= c) r -= c, m >>= 4, pos += 4;
  c = __popc(m & 0x3u);
  if (r >= c) r -= c, m >>= 2, pos += 2;
  return pos + (r >= (int)(m & 1u) ? 1 : 0);
}

__device__ __forceinline__ uint32_t pack_event(int x, int y, bool neg) {
  return (uint32_t)x | ((uint32_t)y << 16) | (neg ? 0x80000000u : 0u);
}

}  // namespace

// ------------------------------------------------------------ segments
// Timestamps of every (pair, link) — chain_events gives each link its later
// frame's stamp, sub_interval_end for the interpolated ones — grouped into
// runs of equal value (finalize's stable_sort, simulate.cpp:36-40, only ever
// reorders inside such a run).  One block; flags + block scan.
__global__ void __launch_bounds__(1024) segments_kernel(SegParams p) {
  __shared__ int s_warp[32];
  const int L = p.d.n_links, G = L * p.n_pairs;
  int carry = 0;
  for (int g0 = 0; g0 < G; g0 += blockDim.x) {
    const int g = g0 + threadIdx.x;
    int64_t t = 0, tp = 0;
    int start = 0;
    if (g < G) {
      const int i = g / L, l = g - i * L;
      auto stamp = [&](int pair, int link) {
        const int k = p.d.start + (link + 1) * p.d.step;
        return k == p.n_interp + 1 ? p.ts[pair + 1]
                                   : sub_interval_end(p.ts[pair], p.ts[pair + 1], k, p.n_interp + 1);
      };
      t = stamp(i, l);
      if (g == 0) {
        start = 1;
      } else {
        const int gi = (g - 1) / L;
        tp = stamp(gi, g - 1 - gi * L);
        start = t != tp;
      }
    }
    int total;
    const int excl = block_exclusive_scan(start, s_warp, total);
    if (g < G && start) {
      const int s = carry + excl;
      p.seg.seg_first[s] = g;
      p.seg.seg_t[s] = t;
    }
    carry += total;
    __syncthreads();
  }
  // run lengths
  for (int s = threadIdx.x; s < carry; s += blockDim.x) {
    const int next = s + 1 < carry ? p.seg.seg_first[s + 1] : G;
    p.seg.seg_nlinks[s] = next - p.seg.seg_first[s];
  }
  if (threadIdx.x == 0) *p.seg.n_segs = carry;
}

// ------------------------------------------------------------ chain kernel
//
// One warp = 32-pixel words of one row, kW words in flight.  For every pair of
// the launch (in stream order, so the log reference state stays in
// registers) and every link of its chain, the warp evaluates the reference
// rule per lane (difference_frame + threshold_events_into, core.cpp:5-46, or
// the log rule of DESIGN.md §3), ballots the crossings and lane 0 stores the
// (pos, neg) masks.  Interpolated values of up to kB links are computed
// before they are chained, so their gathers overlap.  Per-(link, block)
// event counts go to counts[g][block].
template <class Prov, bool kLog, bool kMag, int kW, int kB, int kMinBlocks>
__global__ void __launch_bounds__(256, kMinBlocks) chain_kernel(ChainParams p) {
  extern __shared__ uint32_t s_cnt[];  // [n_pairs * L] event counts of this block
  __shared__ float s_lut[256];
  const int L = p.d.n_links;
  const int G = L * p.n_pairs;
  for (int i = threadIdx.x; i < G; i += blockDim.x) s_cnt[i] = 0;
  if (kLog) s_lut[threadIdx.x] = p.lut[threadIdx.x];
  __syncthreads();
  const int b = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t wbeg = (int64_t)b * p.words_per_block;
  const int64_t wend = min(wbeg + p.words_per_block, p.n_words);
  for (int64_t w0 = wbeg + warp; w0 < wend; w0 += kWarpsPerBlock * kW) {
    PixelCtx c[kW];
    int64_t wi[kW];
    bool have[kW];
    float ref[kW];
#pragma unroll
    for (int q = 0; q < kW; ++q) {
      wi[q] = w0 + q * kWarpsPerBlock;
      have[q] = wi[q] < wend;
      const int64_t ww = have[q] ? wi[q] : w0;
      const int row = (int)((uint32_t)ww / (uint32_t)p.wpr);
      const int x = (int)(ww - (int64_t)row * p.wpr) * 32 + lane;
      c[q].valid = have[q] && x < p.w;
      c[q].x = x < p.w ? x : p.w - 1;
      c[q].y = p.row0 + row;
      c[q].pix = (size_t)c[q].y * p.w + c[q].x;
      c[q].xf = (float)c[q].x;
      c[q].yf = (float)c[q].y;
      if (kLog) ref[q] = p.ref[c[q].pix];
    }
    for (int i = 0; i < p.n_pairs; ++i) {
      const PairCtx pc = pair_ctx(p, i);
      const int gbase = i * L;
      if (pc.skip) {
        if (lane == 0)
          for (int l = 0; l < L; ++l)
#pragma unroll
            for (int q = 0; q < kW; ++q)
              if (have[q]) {
                EVSIM_CHECK((size_t)(gbase + l) * p.n_words + wi[q] < p.masks_cap, "chain mask store");
                p.masks[(size_t)(gbase + l) * p.n_words + wi[q]] = make_uint2(0u, 0u);
              }
        continue;
      }
      Prov prov[kW];
      int before[kW];
#pragma unroll
      for (int q = 0; q < kW; ++q) {
        prov[q].init(p, pc, c[q]);
        if (!kLog) before[q] = frame_value(p, prov[q], pc, c[q], p.d.start);
      }
      for (int l0 = 0; l0 < L; l0 += kB) {
        int vals[kW][kB];
#pragma unroll
        for (int j = 0; j < kB; ++j)
#pragma unroll
          for (int q = 0; q < kW; ++q)
            vals[q][j] = (l0 + j < L) ? frame_value(p, prov[q], pc, c[q], p.d.start + (l0 + j + 1) * p.d.step) : 0;
#pragma unroll
        for (int j = 0; j < kB; ++j) {
          const int l = l0 + j;
          if (l >= L) break;
          const int g = gbase + l;
#pragma unroll
          for (int q = 0; q < kW; ++q) {
            const int val = vals[q][j];
            bool pos, neg;
            int mult = 1;
            if (kLog) {
              const float lk = s_lut[val];
              const float dd = fsub(lk, ref[q]);
              pos = dd > p.c_pos_log;
              neg = !pos && dd < p.c_neg_log;
              if (kMag && (pos || neg)) mult = (int)floorf(__fdiv_rn(dd, pos ? p.c_pos_log : p.c_neg_log));
              if ((pos || neg) && c[q].valid) ref[q] = lk;
            } else {
              const int v = val - before[q];  // difference_frame, core.cpp:14-15
              pos = v > p.c_pos;              // threshold_events_into, core.cpp:31-43
              neg = !pos && v < p.c_neg;
              if (kMag && (pos || neg)) mult = pos ? v / p.c_pos : v / p.c_neg;
              before[q] = val;
            }
            pos = pos && c[q].valid;
            neg = neg && c[q].valid;
            const unsigned bp = __ballot_sync(kFull, pos);
            const unsigned bn = __ballot_sync(kFull, neg);
            if (!have[q]) continue;
            EVSIM_CHECK((size_t)g * p.n_words + wi[q] < p.masks_cap, "chain mask store");
            if (lane == 0) p.masks[(size_t)g * p.n_words + wi[q]] = make_uint2(bp, bn);
            if (kMag) {
              const int m = (pos || neg) ? mult : 0;
              p.mcount[(size_t)g * p.n_words * 32 + wi[q] * 32 + lane] = (uint16_t)m;
              int s = m;
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
              if (lane == 0) {
                p.wcount[(size_t)g * p.n_words + wi[q]] = (uint32_t)s;
                if (s) atomicAdd(&s_cnt[g], (uint32_t)s);
              }
            } else if (lane == 0 && (bp | bn)) {
              atomicAdd(&s_cnt[g], (uint32_t)(__popc(bp) + __popc(bn)));
            }
          }
        }
      }
#pragma unroll
      for (int q = 0; q < kW; ++q)
        if (c[q].valid) prov[q].finish(p, pc, c[q]);
    }
    if (kLog) {
#pragma unroll
      for (int q = 0; q < kW; ++q)
        if (c[q].valid) p.ref[c[q].pix] = ref[q];
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < G; i += blockDim.x) {
    EVSIM_CHECK((size_t)i * p.n_blocks + b < p.counts_cap, "chain count store");
    p.counts[(size_t)i * p.n_blocks + b] = s_cnt[i];
  }
}

// ------------------------------------------------------------ dense chain kernel
//
// chain_kernel specialised for the dense provider on our own (always finite)
// patch-grid flow — the hot loop of dense mode.  Same outputs; differences:
//  * the links into chain frames 1..N run in straight-line batches of kB
//    links x kW words: both bilinear samples of a frame as fp32x2 pairs, the
//    clamps skipped when the whole warp's flow provably stays inside the
//    frame, lround() decided by a bounded fp32 estimate (the rare lanes it
//    cannot decide are recomputed exactly, warp-uniformly, after the batch);
//  * per-frame constants in shared memory, ring slots advanced incrementally.

// Rounded blend of chain frame k (simulate.cpp:108-116) at one pixel.
//   X = x + (-fwd, bwd) * u, Y likewise: (prev sample, curr sample) as lanes.
// The truncations use the magic 2^23 for X and my = 2^23 + m_y for Y
// (ChainParams::magic_y); the gather index TY_bits * w + TX_bits then equals
// y * w + x + qshift without wrapping, and qp / qc come pre-shifted by
// -qshift elements, so the index costs one IMAD.
// The blend weights are two of the position constants: kc = (-(float)alpha,
// (float)(1 - alpha), (float)oma, (float)alpha) holds oma_f = kc.y and
// alpha_f = -kc.x bit for bit (host: evsim_gpu.cu allocate()), so a link
// needs one 8-byte constant load, not two.
template <bool kClamp>
__device__ __forceinline__ int dense_fast(const uint32_t* __restrict__ qp, const uint32_t* __restrict__ qc,
                                          uint32_t w, float my, float wm, float hm, float xf, float yf,
                                          float u, float v, float4 kc, unsigned& bad, unsigned bit) {
  const f32x2 NB = pk2(kc.x, kc.y);
  f32x2 X = affine2_est(xf, NB, u), Y = affine2_est(yf, NB, v);
  if (kClamp) {
    X = pk2(fminf(fmaxf(lo2(X), 0.0f), wm), fminf(fmaxf(hi2(X), 0.0f), wm));
    Y = pk2(fminf(fmaxf(lo2(Y), 0.0f), hm), fminf(fmaxf(hi2(Y), 0.0f), hm));
  }
  const f32x2 C23 = pk2(8388608.0f, 8388608.0f);
  const f32x2 CY = pk2(my, my);
  const f32x2 TX = add2_rz(X, C23), TY = add2_rz(Y, CY);  // magic + trunc
  const f32x2 FX = sub2(X, sub2(TX, C23)), FY = sub2(Y, sub2(TY, CY));
  const uint32_t ia = __float_as_uint(lo2(TY)) * w + __float_as_uint(lo2(TX));
  const uint32_t ib = __float_as_uint(hi2(TY)) * w + __float_as_uint(hi2(TX));
  const uint32_t va = __ldg(qp + ia), vb = __ldg(qc + ib);
  // taps as 2^23 + byte (PRMT); differences of biased taps are exact
  const f32x2 B00 = pk2(__uint_as_float(__byte_perm(va, 0x4B000000u, 0x7540)),
                        __uint_as_float(__byte_perm(vb, 0x4B000000u, 0x7540)));
  const f32x2 B10 = pk2(__uint_as_float(__byte_perm(va, 0x4B000000u, 0x7541)),
                        __uint_as_float(__byte_perm(vb, 0x4B000000u, 0x7541)));
  const f32x2 B01 = pk2(__uint_as_float(__byte_perm(va, 0x4B000000u, 0x7542)),
                        __uint_as_float(__byte_perm(vb, 0x4B000000u, 0x7542)));
  const f32x2 B11 = pk2(__uint_as_float(__byte_perm(va, 0x4B000000u, 0x7543)),
                        __uint_as_float(__byte_perm(vb, 0x4B000000u, 0x7543)));
  const f32x2 top = lerpd2_est(sub2(B00, C23), sub2(B10, B00), FX);
  const f32x2 bot = lerpd2_est(sub2(B01, C23), sub2(B11, B01), FX);
  const f32x2 S = lerp2_est(top, bot, FY);
  // s = RN64(RN64(oma*fp) + RN64(alpha*fc)); e below satisfies |e - s| < 6.2e-5
  // (see DenseProvider::interp), RN(e + c) adds < 1.6e-5.  If
  // floor(e + 0.5 -/+ 2e-4) agree, that floor is lround(s) = floor(s + 0.5).
  const float e = __fmaf_rn(kc.y, lo2(S), __fmul_rn(-kc.x, hi2(S)));  // (oma_f = kc.y, alpha_f = -kc.x)
  const f32x2 T = add2_rz(add2(pk2(e, e), pk2(0.5f - 2e-4f, 0.5f + 2e-4f)), C23);
  if (__float_as_uint(lo2(T)) != __float_as_uint(hi2(T))) bad |= bit;
  return __float_as_int(hi2(T));  // kVB + value (the bias folds into the LUT address / cancels in differences)
}

// dense_fast on the fp32 lerp quads of the frames — with dx = a10 - a00,
// dy = a01 - a00, dxy = (a11 - a01) - (a10 - a00), stored relative to the
// tap column (see below) — one 16-byte gather per
// sample, no byte unpack, and each sample as three FFMA — top = a00 + fx*dx,
// (bottom - top) = dy + fx*dxy (exactly the difference of the two row lerps,
// |.| <= 255, one rounding), s = top + fy*(bottom - top) — an estimate, like
// e.  The positions X, Y and their splits are the reference's exactly (as
// above).  Bound (u = 2^-17, half an ulp in [128, 256)): the reference's fp32
// sample (simulate.cpp:10-26) is within 5u of the exact bilinear value (2u
// per row lerp, + the rounded difference, product and sum), this one within
// 3u (u for top, u for the difference, fy <= 1, u for s), so |fp - fp_ref| <= 8u
// = 6.1e-5, the same for fc; with the fp32 weights (|oma_f - oma| <= 2^-25,
// oma + alpha = 1) and e's two fp32 roundings, |e - s| <= 255 * 2^-24 + 8u
// + 2u < 9.2e-5, and RN(e + 0.5 -/+ 2e-4) adds < 1.6e-5: inside the 2e-4
// decision margin, so a decided lane rounds exactly like the reference.
template <bool kClamp>
__device__ __forceinline__ int dense_fast(const float4* __restrict__ qp, const float4* __restrict__ qc,
                                          uint32_t w, float my, float wm, float hm, float xf, float yf,
                                          float u, float v, float4 kc, unsigned& bad, unsigned bit) {
  const f32x2 NB = pk2(kc.x, kc.y);
  f32x2 X = affine2_est(xf, NB, u), Y = affine2_est(yf, NB, v);
  if (kClamp) {
    X = pk2(fminf(fmaxf(lo2(X), 0.0f), wm), fminf(fmaxf(hi2(X), 0.0f), wm));
    Y = pk2(fminf(fmaxf(lo2(Y), 0.0f), hm), fminf(fmaxf(hi2(Y), 0.0f), hm));
  }
  const f32x2 C23 = pk2(8388608.0f, 8388608.0f);
  const f32x2 CY = pk2(my, my);
  const f32x2 TX = add2_rz(X, C23), TY = add2_rz(Y, CY);  // magic + trunc
  const f32x2 FY = sub2(Y, sub2(TY, CY));
  const uint32_t ia = __float_as_uint(lo2(TY)) * w + __float_as_uint(lo2(TX));
  const uint32_t ib = __float_as_uint(hi2(TY)) * w + __float_as_uint(hi2(TX));
  // quad of tap column x0 = (a00 - x0*dx, dx, dy - x0*dxy, dxy), exact integers
  // below 2^24 (kLerpQuadMaxW): the fma forms X*dx + (a00 - x0*dx) exactly
  // before its one rounding, and X - x0 is the x fraction exactly, so
  // top = RN(a00 + fx*dx) and bottom - top = RN(dy + fx*dxy) bit for bit —
  // without ever forming fx
  const float4 A = __ldg(qp + ia), B = __ldg(qc + ib);
  const float ta = __fmaf_rn(lo2(X), A.y, A.x), da = __fmaf_rn(lo2(X), A.w, A.z);
  const float tb = __fmaf_rn(hi2(X), B.y, B.x), db = __fmaf_rn(hi2(X), B.w, B.z);
  const float sa = __fmaf_rn(lo2(FY), da, ta);
  const float sb = __fmaf_rn(hi2(FY), db, tb);
  const float e = __fmaf_rn(kc.y, sa, __fmul_rn(-kc.x, sb));  // (oma_f = kc.y, alpha_f = -kc.x)
  const f32x2 T = add2_rz(add2(pk2(e, e), pk2(0.5f - 2e-4f, 0.5f + 2e-4f)), C23);
  if (__float_as_uint(lo2(T)) != __float_as_uint(hi2(T))) bad |= bit;
  return __float_as_int(hi2(T));
}

// dense_fast on bf16 lerp quads: per pixel two words (a00 | (a10 - a00) << 16,
// a01 | (a11 - a01) << 16) of bf16 values — integers |v| <= 255 have at most
// 8 significant bits, so bf16 holds them exactly and a bf16 is the high half
// of the fp32 with the same value.  8 bytes per gather; each value back to
// fp32 by one shift or mask; then the same FFMA lerps and bound as above.
template <bool kClamp>
__device__ __forceinline__ int dense_fast(const uint2* __restrict__ qp, const uint2* __restrict__ qc,
                                          uint32_t w, float my, float wm, float hm, float xf, float yf,
                                          float u, float v, float4 kc, unsigned& bad, unsigned bit) {
  const f32x2 NB = pk2(kc.x, kc.y);
  f32x2 X = affine2_est(xf, NB, u), Y = affine2_est(yf, NB, v);
  if (kClamp) {
    X = pk2(fminf(fmaxf(lo2(X), 0.0f), wm), fminf(fmaxf(hi2(X), 0.0f), wm));
    Y = pk2(fminf(fmaxf(lo2(Y), 0.0f), hm), fminf(fmaxf(hi2(Y), 0.0f), hm));
  }
  const f32x2 C23 = pk2(8388608.0f, 8388608.0f);
  const f32x2 CY = pk2(my, my);
  const f32x2 TX = add2_rz(X, C23), TY = add2_rz(Y, CY);  // magic + trunc
  const f32x2 FX = sub2(X, sub2(TX, C23)), FY = sub2(Y, sub2(TY, CY));
  const uint32_t ia = __float_as_uint(lo2(TY)) * w + __float_as_uint(lo2(TX));
  const uint32_t ib = __float_as_uint(hi2(TY)) * w + __float_as_uint(hi2(TX));
  const uint2 A = __ldg(qp + ia), B = __ldg(qc + ib);
  auto lo16 = [](uint32_t x) { return __uint_as_float(x << 16); };
  auto hi16 = [](uint32_t x) { return __uint_as_float(x & 0xFFFF0000u); };
  const float ta = __fmaf_rn(lo2(FX), hi16(A.x), lo16(A.x)), ba = __fmaf_rn(lo2(FX), hi16(A.y), lo16(A.y));
  const float tb = __fmaf_rn(hi2(FX), hi16(B.x), lo16(B.x)), bb = __fmaf_rn(hi2(FX), hi16(B.y), lo16(B.y));
  const float sa = __fmaf_rn(lo2(FY), __fsub_rn(ba, ta), ta);
  const float sb = __fmaf_rn(hi2(FY), __fsub_rn(bb, tb), tb);
  const float e = __fmaf_rn(kc.y, sa, __fmul_rn(-kc.x, sb));  // (oma_f = kc.y, alpha_f = -kc.x)
  const f32x2 T = add2_rz(add2(pk2(e, e), pk2(0.5f - 2e-4f, 0.5f + 2e-4f)), C23);
  if (__float_as_uint(lo2(T)) != __float_as_uint(hi2(T))) bad |= bit;
  return __float_as_int(hi2(T));
}

// The exact reference expression for the lanes dense_fast cannot decide.
__device__ __noinline__ int dense_exact(const float2* nfb, const double* oma, const double* alpha,
                                        const uint32_t* qp, const uint32_t* qc, int w, int h, float xf, float yf,
                                        float u, float v, int k) {
  const float2 nb = __ldg(nfb + k);
  const f32x2 NB = pk2(nb.x, nb.y);
  const f32x2 S = sample_quad_pair(qp, qc, w, h, affine2(xf, NB, u), affine2(yf, NB, v));
  const double blend = dadd(dmul(__ldg(oma + k), (double)lo2(S)), dmul(__ldg(alpha + k), (double)hi2(S)));
  return lround_pos_fast(blend);
}

// chain values in the dense kernel carry this bias: the fp32 bits of 2^23 + v
constexpr int kVB = kChainBias;

struct DenseWord {
  bool have, valid;
  uint32_t wi;  // word index (n_words < 2^32)
  int x, y;
  uint32_t pix;
  float xf, yf;
  float u, v;
};

// One link of the chain at one word: the reference rule and its ballots.
// ev = the word's events of this link (crossings, or magnitudes).
template <bool kLog, bool kMag>
__device__ __forceinline__ uint2 link_rule(const ChainParams& p, const float* s_lut, int g, const DenseWord& c,
                                           int lane, int val, float& ref, int& before, uint32_t& ev) {
  bool pos, neg;
  int mult = 1;
  if (kLog) {
    const float lk = s_lut[val];
    const float dd = fsub(lk, ref);
    pos = dd > p.c_pos_log;
    neg = !pos && dd < p.c_neg_log;
    if (kMag && (pos || neg)) mult = (int)floorf(__fdiv_rn(dd, pos ? p.c_pos_log : p.c_neg_log));
    if ((pos || neg) && c.valid) ref = lk;
  } else {
    const int d = val - before;  // difference_frame, core.cpp:14-15
    pos = d > p.c_pos;           // threshold_events_into, core.cpp:31-43
    neg = !pos && d < p.c_neg;
    if (kMag && (pos || neg)) mult = pos ? d / p.c_pos : d / p.c_neg;
    before = val;
  }
  pos = pos && c.valid;
  neg = neg && c.valid;
  const unsigned bp = __ballot_sync(kFull, pos);
  const unsigned bn = __ballot_sync(kFull, neg);
  if (kMag) {
    const int m = (pos || neg) ? mult : 0;
    if (c.have) p.mcount[(size_t)g * p.n_words * 32 + c.wi * 32 + lane] = (uint16_t)m;
    int sm = m;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sm += __shfl_xor_sync(kFull, sm, o);
    ev = (uint32_t)sm;
  } else {
    ev = (uint32_t)__popc(bp | bn);  // a pixel crosses one way or not at all
  }
  return make_uint2(bp, bn);
}

// link_rule for single mode in the dense kernel, on biased values: the log
// rule's LUT read folds the bias into the shared-window base (lut_b); lanes
// past the row end hold ref = NaN (no comparison holds, ref never changes),
// so validity needs no per-link test in log mode.  Event counts are taken
// from the masks when they are flushed.
template <bool kLog>
__device__ __forceinline__ uint2 dense_rule(const ChainParams& p, uint32_t lut_b, const DenseWord& c, int val,
                                            float& ref, int& before) {
  bool pos, neg;
  if (kLog) {
    float lk;
    asm("ld.shared.f32 %0, [%1];" : "=f"(lk) : "r"(lut_b + ((uint32_t)val << 2)));
    const float dd = fsub(lk, ref);
    pos = dd > p.c_pos_log;  // c_pos_log > 0 > c_neg_log (validated): exclusive
    neg = dd < p.c_neg_log;
    if (pos || neg) ref = lk;
  } else {
    const int d = val - before;  // difference_frame, core.cpp:14-15 (biases cancel)
    pos = d > p.c_pos && c.valid;  // threshold_events_into, core.cpp:31-43
    neg = d < p.c_neg && c.valid;
    before = val;
  }
  return make_uint2(__ballot_sync(kFull, pos), __ballot_sync(kFull, neg));
}

// dense_rule for log single mode as level thresholds: the
// reference state is always a LUT level L[r] (init_ref sets L(frame0), an
// event sets L(v)), and fsub(L[v], L[r]) is monotone in v, so d > c_pos <=>
// v > hi[r] and d < c_neg <=> v < lo[r] (host table lthr, biased like val).
// The lane keeps its level's (hi, lo) and value; only lanes that fired
// reload them (one 8-byte LDS) — no LUT read and no fp32 subtraction per
// link.  Padding lanes hold (INT_MAX, INT_MIN): they never fire.
__device__ __forceinline__ uint2 dense_rule_th(uint32_t th_b, int val, int& thh, int& thl, int& vr) {
  const bool pos = val > thh, neg = val < thl;
  const unsigned bp = __ballot_sync(kFull, pos), bn = __ballot_sync(kFull, neg);
  if (pos || neg) {
    asm("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(thh), "=r"(thl) : "r"(th_b + ((uint32_t)val << 3)));
    vr = val;
  }
  return make_uint2(bp, bn);
}

template <int kW, int kNB, bool kClamp, int kBM, class Q>
__device__ __forceinline__ unsigned dense_batch(const ChainParams& p, const Q* qp, const Q* qc,
                                                uint32_t w, float my, float wm, float hm, const DenseWord* c,
                                                int k0, int (&vals)[kW][kBM]) {
  unsigned bad = 0;
#pragma unroll
  for (int j = 0; j < kNB; ++j) {
    const float4 kc = p.kcp[k0 + j];
#pragma unroll
    for (int q = 0; q < kW; ++q)
      vals[q][j] = dense_fast<kClamp>(qp, qc, w, my, wm, hm, c[q].xf, c[q].yf, c[q].u, c[q].v, kc, bad,
                                      1u << (q * kBM + j));
  }
  return bad;
}

// kW words per warp (1 on small frames: finer tasks, 4 blocks per SM; 2 on
// large ones), kB links per batch (4, or 5 when it tiles the interior links)
template <bool kLog, bool kMag, int kB, int kW, int kMinB, int kQ>
__global__ void __launch_bounds__(256, kMinB) chain_dense_kernel(ChainParams p) {
  // gather image: 0 = u8 quads, 1 = fp32 lerp quads, 2 = bf16 lerp quads
  using Q = std::conditional_t<kQ == 1, float4, std::conditional_t<kQ == 2, uint2, uint32_t>>;
  constexpr bool kTh = kLog && !kMag;  // log single mode: level thresholds (dense_rule_th)
  extern __shared__ float4 s_dyn4[];
  __shared__ float s_lut[256];
  __shared__ int2 s_th[kTh ? 256 : 1];
  constexpr int kStage = 32 + kB;  // staged links of a warp: < 32 before a batch of kB
  __shared__ uint2 s_stm[kWarpsPerBlock][kW][kStage];
  __shared__ uint32_t s_stc[kMag ? kWarpsPerBlock : 1][kMag ? kStage : 1];
  __shared__ uint32_t s_stw[kMag ? kWarpsPerBlock : 1][kW][kMag ? kStage : 1];
  const int L = p.d.n_links, G = L * p.n_pairs, N = p.n_interp;
  // (the chain constants come from the kernel parameters, p.kcp)
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_dyn4 + N + 2);  // [G]
  for (int i = threadIdx.x; i < G; i += blockDim.x) s_cnt[i] = 0;
  if (kLog) s_lut[threadIdx.x] = p.lut[threadIdx.x];
  if (kTh) s_th[threadIdx.x] = make_int2(p.lthr[threadIdx.x].x, p.lthr[threadIdx.x].y);  // (hi, lo) of level threadIdx.x
  __syncthreads();
  const int b = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t w = (uint32_t)p.w;
  const float wm = (float)(p.w - 1), hm = (float)(p.h - 1);
  const float my = p.magic_y;
  const uint32_t lut_b = pin((uint32_t)__cvta_generic_to_shared(s_lut) - ((uint32_t)kVB << 2));
  const uint32_t th_b = pin((uint32_t)__cvta_generic_to_shared(s_th) - ((uint32_t)kVB << 3));
  // link l joins chain frames start + l and start + l + 1; the first n_int
  // links end in an interpolated frame (k <= N), a last one (endpoints) in curr
  const int kfirst = p.d.start + 1;
  const int n_int = min(L, N - p.d.start);
  const int64_t wbeg = (int64_t)b * p.words_per_block;
  const int64_t wend = min(wbeg + p.words_per_block, p.n_words);
  for (int64_t w0 = wbeg + warp; w0 < wend; w0 += kWarpsPerBlock * kW) {
    DenseWord c[kW];
    float ref[kW];
    int before[kW];
    int thh[kW], thl[kW], vr[kW];  // kTh: the level's (hi, lo) and biased value
#pragma unroll
    for (int q = 0; q < kW; ++q) {
      const int64_t wq = w0 + q * kWarpsPerBlock;
      c[q].have = wq < wend;
      c[q].wi = (uint32_t)wq;
      const int64_t ww = c[q].have ? wq : w0;
      const int row = (int)((uint32_t)ww / (uint32_t)p.wpr);
      const int x = (int)(ww - (int64_t)row * p.wpr) * 32 + lane;
      c[q].valid = c[q].have && x < p.w;
      c[q].x = x < p.w ? x : p.w - 1;
      c[q].y = p.row0 + row;
      c[q].pix = (uint32_t)c[q].y * w + (uint32_t)c[q].x;
      c[q].xf = (float)c[q].x;
      c[q].yf = (float)c[q].y;
      ref[q] = kLog ? (c[q].valid ? p.ref[c[q].pix] : __int_as_float(0x7FC00000)) : 0.0f;
      before[q] = 0;
      if constexpr (kTh) {
        thh[q] = INT_MAX;
        thl[q] = INT_MIN;
        vr[q] = kVB;
        if (c[q].valid) {
          // the level r with L[r] == ref (ref is always a LUT value): the
          // largest r with L[r] <= ref, L strictly increasing
          int r = 0;
#pragma unroll
          for (int st = 128; st >= 1; st >>= 1)
            if (s_lut[r + st] <= ref[q]) r += st;
          const int2 t = s_th[r];
          thh[q] = t.x;
          thl[q] = t.y;
          vr[q] = kVB + r;
        }
      }
    }
    int sp = p.r0 % p.R;
    for (int i = 0; i < p.n_pairs; ++i) {
      const int sc = sp + 1 == p.R ? 0 : sp + 1;
      const uint32_t* qp = p.quads.at(sp);
      const uint32_t* qc = p.quads.at(sc);
      const uint32_t* qbp = reinterpret_cast<const uint32_t*>(reinterpret_cast<uintptr_t>(qp) - 4ull * p.qshift);
      const uint32_t* qbc = reinterpret_cast<const uint32_t*>(reinterpret_cast<uintptr_t>(qc) - 4ull * p.qshift);
      // the gathers' rings (fp32 lerp quads or u8 quads), pre-shifted by -qshift elements
      const Q* gbp;
      const Q* gbc;
      if constexpr (kQ == 1) {
        gbp = reinterpret_cast<const float4*>(reinterpret_cast<uintptr_t>(p.quadf.at(sp)) - 16ull * p.qshift);
        gbc = reinterpret_cast<const float4*>(reinterpret_cast<uintptr_t>(p.quadf.at(sc)) - 16ull * p.qshift);
      } else if constexpr (kQ == 2) {
        gbp = reinterpret_cast<const uint2*>(reinterpret_cast<uintptr_t>(p.quadh.at(sp)) - 8ull * p.qshift);
        gbc = reinterpret_cast<const uint2*>(reinterpret_cast<uintptr_t>(p.quadh.at(sc)) - 8ull * p.qshift);
      } else {
        gbp = qbp;
        gbc = qbc;
      }
      PairCtx pc{};
      pc.pu = p.g0.pu + (size_t)i * p.g0.pair_stride;
      pc.pv = p.g0.pv + (size_t)i * p.g0.pair_stride;
      bool safe = true;
#pragma unroll
      for (int q = 0; q < kW; ++q) {
        PixelCtx pxc;
        pxc.x = c[q].x;
        pxc.y = c[q].y;
        DenseProvider<false> prov;
        prov.init(p, pc, pxc);
        c[q].u = prov.u;
        c[q].v = prov.v;
        // every sample x + s*u, |s| <= 1, stays in [0, w-1] (rounding is
        // monotone and the bounds are representable): no clamp needed
        safe = safe && fabsf(prov.u) <= fminf(c[q].xf, wm - c[q].xf) && fabsf(prov.v) <= fminf(c[q].yf, hm - c[q].yf);
        if (!kLog)
          before[q] = kVB + (p.d.start == 0 ? (int)p.frames.at(sp)[c[q].pix]
                                            : dense_exact(p.nfb, p.oma, p.alpha, qp, qc, p.w, p.h, c[q].xf, c[q].yf,
                                                          prov.u, prov.v, 1));
      }
      safe = __all_sync(kFull, safe);
      const int gbase = i * L;
      // lane 0 stages each link's masks (warp-uniform ballots) and event count
      // in shared memory; once 32 or more links are staged (checked per batch)
      // lane j stores / adds staged link j
      int fbase = 0;
      auto step = [&](int l, int q, int val) {
        if (kMag) {
          uint32_t ev;
          int bv = before[q] - kVB;
          const uint2 m = link_rule<kLog, kMag>(p, s_lut, gbase + l, c[q], lane, val - kVB, ref[q], bv, ev);
          before[q] = bv + kVB;
          if (lane == 0) {
            s_stm[warp][q][l - fbase] = m;
            s_stw[warp][q][l - fbase] = ev;
            if (q == 0) s_stc[warp][l - fbase] = ev;
            else s_stc[warp][l - fbase] += ev;
          }
        } else if constexpr (kTh) {
          const uint2 m = dense_rule_th(th_b, val, thh[q], thl[q], vr[q]);
          if (lane == 0) s_stm[warp][q][l - fbase] = m;
        } else {
          const uint2 m = dense_rule<kLog>(p, lut_b, c[q], val, ref[q], before[q]);
          if (lane == 0) s_stm[warp][q][l - fbase] = m;
        }
      };
      auto flush = [&](int lend, bool force) {
        const int n = lend - fbase;
        if (n < 32 && !force) return;
        __syncwarp();
        for (int j = lane; j < n; j += 32) {
          const int g = gbase + fbase + j;
          uint32_t cnt = 0;
#pragma unroll
          for (int q = 0; q < kW; ++q) {
            if (!c[q].have) continue;
            const uint2 m = s_stm[warp][q][j];
            EVSIM_CHECK((size_t)g * p.n_words + c[q].wi < p.masks_cap, "dense chain mask store");
            p.masks[(size_t)g * p.n_words + c[q].wi] = m;
            if (kMag) p.wcount[(size_t)g * p.n_words + c[q].wi] = s_stw[warp][q][j];
            else cnt += __popc(m.x | m.y);  // a pixel crosses one way or not at all
          }
          if (kMag) cnt = s_stc[warp][j];
          if (cnt) atomicAdd(&s_cnt[g], cnt);
        }
        __syncwarp();
        fbase = lend;
      };
      int l0 = 0;
      for (; l0 < n_int; l0 += kB) {
        const int nb = min(kB, n_int - l0);
        int vals[kW][kB];
        unsigned bad;
        if (nb == kB) {
          bad = safe ? dense_batch<kW, kB, false>(p, gbp, gbc, w, my, wm, hm, c, kfirst + l0, vals)
                     : dense_batch<kW, kB, true>(p, gbp, gbc, w, my, wm, hm, c, kfirst + l0, vals);
        } else {
          bad = 0;
          for (int j = 0; j < nb; ++j) {
            int v1[kW][kB];
            bad |= (safe ? dense_batch<kW, 1, false>(p, gbp, gbc, w, my, wm, hm, c, kfirst + l0 + j, v1)
                         : dense_batch<kW, 1, true>(p, gbp, gbc, w, my, wm, hm, c, kfirst + l0 + j, v1))
                   << j;
#pragma unroll
            for (int q = 0; q < kW; ++q)
#pragma unroll
              for (int jj = 0; jj < kB; ++jj)
                if (jj == j) vals[q][jj] = v1[q][0];
          }
        }
        if (__any_sync(kFull, bad != 0u)) {
#pragma unroll
          for (int q = 0; q < kW; ++q)
#pragma unroll
            for (int j = 0; j < kB; ++j)
              if ((bad >> (q * kB + j)) & 1u)
                vals[q][j] = kVB + dense_exact(p.nfb, p.oma, p.alpha, qp, qc, p.w, p.h, c[q].xf, c[q].yf, c[q].u,
                                             c[q].v, kfirst + l0 + j);
        }
        if (nb == kB) {
#pragma unroll
          for (int j = 0; j < kB; ++j)
#pragma unroll
            for (int q = 0; q < kW; ++q) step(l0 + j, q, vals[q][j]);
        } else {
#pragma unroll
          for (int j = 0; j < kB; ++j) {
            if (j >= nb) break;
#pragma unroll
            for (int q = 0; q < kW; ++q) step(l0 + j, q, vals[q][j]);
          }
        }
        flush(l0 + nb, false);
      }
      if (n_int < L) {  // the link into curr (include_endpoints)
        const uint8_t* curr = p.frames.at(sc);
#pragma unroll
        for (int q = 0; q < kW; ++q) step(L - 1, q, kVB + (int)curr[c[q].pix]);
      }
      flush(L, true);
      sp = sc;
    }
    if (kLog) {
#pragma unroll
      for (int q = 0; q < kW; ++q)
        if (c[q].valid) p.ref[c[q].pix] = kTh ? s_lut[vr[q] - kVB] : ref[q];
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < G; i += blockDim.x) {
    EVSIM_CHECK((size_t)i * p.n_blocks + b < p.counts_cap, "chain count store");
    p.counts[(size_t)i * p.n_blocks + b] = s_cnt[i];
  }
}

// ------------------------------------------------------------ difference_only chain
//
// chain_kernel specialised for difference_only (N = 0, one link per pair:
// prev -> curr, simulate.cpp:322-327 -> core.cpp:5-46) in single mode.  A
// warp owns one 32-pixel word and walks the launch's pairs in order (the log
// state / the previous value stay in registers); the frame bytes of kP pairs
// are loaded together before they are chained, so kP loads are in flight per
// warp — the chain is a pure stream over the frames.  The log rule uses the
// per-level thresholds (dense_rule_th), the linear one the biased-value
// difference; masks are staged per warp and stored 32 links at a time, as in
// the dense chain.
template <bool kLog, int kP>
__global__ void __launch_bounds__(256) chain_diff_kernel(ChainParams p) {
  extern __shared__ uint32_t s_cnt[];  // [n_pairs] event counts of this block
  __shared__ float s_lut[kLog ? 256 : 1];
  __shared__ int2 s_th[kLog ? 256 : 1];
  constexpr int kStage = 32 + kP;
  __shared__ uint2 s_stm[kWarpsPerBlock][kStage];
  const int G = p.n_pairs;
  for (int i = threadIdx.x; i < G; i += blockDim.x) s_cnt[i] = 0;
  if (kLog) {
    s_lut[threadIdx.x] = p.lut[threadIdx.x];
    s_th[threadIdx.x] = make_int2(p.lthr[threadIdx.x].x, p.lthr[threadIdx.x].y);
  }
  __syncthreads();
  const int b = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t th_b = pin((uint32_t)__cvta_generic_to_shared(s_th) - ((uint32_t)kVB << 3));
  const int64_t wbeg = (int64_t)b * p.words_per_block;
  const int64_t wend = min(wbeg + p.words_per_block, p.n_words);
  for (int64_t wi = wbeg + warp; wi < wend; wi += kWarpsPerBlock) {
    const int row = (int)((uint32_t)wi / (uint32_t)p.wpr);
    const int x = (int)(wi - (int64_t)row * p.wpr) * 32 + lane;
    const bool valid = x < p.w;
    const size_t pix = (size_t)(p.row0 + row) * p.w + (valid ? x : p.w - 1);
    int before = 0, thh = INT_MAX, thl = INT_MIN, vr = kVB;
    int sp = p.r0 % p.R;
    if (kLog) {
      if (valid) {
        const float ref = p.ref[pix];
        int r = 0;  // the level with L[r] == ref (see chain_dense_kernel)
#pragma unroll
        for (int st = 128; st >= 1; st >>= 1)
          if (s_lut[r + st] <= ref) r += st;
        const int2 t = s_th[r];
        thh = t.x;
        thl = t.y;
        vr = kVB + r;
      }
    } else {
      before = kVB + (int)__ldg((p.dcurr ? p.dprev : p.frames.at(sp)) + pix);
    }
    const uint8_t* dc = p.dcurr ? p.dcurr + pix : nullptr;  // direct: pair i's curr at dc + i*P
    int fbase = 0;
    for (int i0 = 0; i0 < G; i0 += kP) {
      int vals[kP];
#pragma unroll
      for (int j = 0; j < kP; ++j) {
        sp = sp + 1 == p.R ? 0 : sp + 1;  // curr of pair i0 + j
        const uint8_t* src = dc ? dc + (size_t)(i0 + j) * p.P : p.frames.at(sp) + pix;
        vals[j] = i0 + j < G ? kVB + (int)__ldg(src) : 0;
      }
#pragma unroll
      for (int j = 0; j < kP; ++j) {
        if (i0 + j >= G) break;
        uint2 m;
        if (kLog) {
          m = dense_rule_th(th_b, vals[j], thh, thl, vr);
        } else {
          const int d = vals[j] - before;  // difference_frame, core.cpp:14-15
          m = make_uint2(__ballot_sync(kFull, d > p.c_pos && valid), __ballot_sync(kFull, d < p.c_neg && valid));
          before = vals[j];
        }
        if (lane == 0) s_stm[warp][i0 + j - fbase] = m;
      }
      const int lend = min(i0 + kP, G);
      if (lend - fbase >= 32 || lend == G) {  // store the staged links' masks
        __syncwarp();
        for (int j = lane; j < lend - fbase; j += 32) {
          const uint2 m = s_stm[warp][j];
          EVSIM_CHECK((size_t)(fbase + j) * p.n_words + wi < p.masks_cap, "diff chain mask store");
          p.masks[(size_t)(fbase + j) * p.n_words + wi] = m;
          const uint32_t cnt = __popc(m.x | m.y);
          if (cnt) atomicAdd(&s_cnt[fbase + j], cnt);
        }
        __syncwarp();
        fbase = lend;
      }
    }
    if (kLog && valid) p.ref[pix] = s_lut[vr - kVB];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < G; i += blockDim.x) {
    EVSIM_CHECK((size_t)i * p.n_blocks + b < p.counts_cap, "chain count store");
    p.counts[(size_t)i * p.n_blocks + b] = s_cnt[i];
  }
}

// ---- TMA-staged form -------------------------------------------------------
// The same chain with the frames staged in shared memory: a block walks its
// words in chunks of kTW (8 warps x kWPW words); for every pair of the
// launch one thread bulk-copies the chunk's rows of the pair's curr frame
// (cp.async.bulk global -> shared, 16-byte aligned range, completion on an
// mbarrier) into a kNB-deep ring of stage buffers, kNB frames ahead of the
// warps, which read their bytes with LDS.  One contiguous copy per (chunk,
// frame) instead of one 32-byte gather per (word, frame): the frames stream
// from HBM in long runs.  Needs 16-byte aligned frames (P % 16 == 0, aligned
// base): chain_diff_tma_ok().
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "fence.proxy.async.shared::cta;\n"
      "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%3], %2;\n"
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

constexpr int kDiffWPW = 8;                           // words per warp per chunk
constexpr int kDiffTW = kWarpsPerBlock * kDiffWPW;   // words per chunk
constexpr int kDiffNB = 4;                            // frames in flight per block
constexpr int kDiffMinB = 4;                          // blocks per SM (64 registers)

template <bool kLog>
__global__ void __launch_bounds__(256, kDiffMinB) chain_diff_tma_kernel(ChainParams p, int stage_bytes) {
  extern __shared__ __align__(128) uint8_t s_raw[];  // [kDiffNB][stage_bytes] frames, then [n_pairs] counts
  __shared__ float s_lut[kLog ? 256 : 1];
  __shared__ int2 s_th[kLog ? 256 : 1];
  __shared__ __align__(8) uint64_t s_bar[kDiffNB];
  __shared__ uint2 s_stm[kWarpsPerBlock][kDiffWPW][32 + 1];
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_raw + (size_t)kDiffNB * stage_bytes);
  const int G = p.n_pairs;
  for (int i = threadIdx.x; i < G; i += blockDim.x) s_cnt[i] = 0;
  if (kLog) {
    s_lut[threadIdx.x] = p.lut[threadIdx.x];
    // (hi, lo) of level threadIdx.x, unbiased: this chain compares raw bytes
    s_th[threadIdx.x] = make_int2(p.lthr[threadIdx.x].x - kVB, p.lthr[threadIdx.x].y - kVB);
  }
  const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(s_bar);
  const uint32_t buf0 = (uint32_t)__cvta_generic_to_shared(s_raw);
  if (threadIdx.x == 0) {
    for (int k = 0; k < kDiffNB; ++k) mbar_init(bar0 + 8 * k, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int b = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t th_b = pin((uint32_t)__cvta_generic_to_shared(s_th));
  // lane 0 stages link (i - fbase)'s masks of word q at st_b + (i - fbase) * 8 + q * kStRow
  constexpr uint32_t kStRow = sizeof(s_stm[0][0]);
  const uint32_t st_b = pin((uint32_t)__cvta_generic_to_shared(&s_stm[warp][0][0]));
  const int64_t wbeg = (int64_t)b * p.words_per_block;
  const int64_t wend = min(wbeg + p.words_per_block, p.n_words);
  const int n_chunks = (int)((wend - wbeg + kDiffTW - 1) / kDiffTW);
  const int64_t total = (int64_t)n_chunks * G;  // (chunk, pair) copies of this block, in order
  // the byte range [a0, a0 + bytes) of chunk c's rows in a frame (16-aligned)
  auto range = [&](int c, size_t& a0, uint32_t& bytes) {
    const int64_t cw0 = wbeg + (int64_t)c * kDiffTW, cw1 = min(cw0 + kDiffTW, wend);
    const size_t r0 = (size_t)(p.row0 + (int)((uint32_t)cw0 / (uint32_t)p.wpr));
    const size_t r1 = (size_t)(p.row0 + (int)((uint32_t)(cw1 - 1) / (uint32_t)p.wpr)) + 1;
    a0 = (r0 * (size_t)p.w) & ~(size_t)15;
    bytes = (uint32_t)((((r1 * (size_t)p.w) + 15) & ~(size_t)15) - a0);
  };
  // producer (thread 0): copy t = (chunk pc, pair pi) into stage t % kDiffNB;
  // its chunk's range and the pair's ring slot advance incrementally
  int64_t pt = 0;
  int pc = 0, pi = 0, pslot = 0;
  size_t pa0 = 0;
  uint32_t pbytes = 0;
  auto issue_next = [&]() {
    if (pi == 0) {
      range(pc, pa0, pbytes);
      pslot = p.r0 + 1;
      while (pslot >= p.R) pslot -= p.R;
    }
    const uint8_t* f = p.dcurr ? p.dcurr + (size_t)pi * p.P : p.frames.at(pslot);
    const int st = (int)(pt & (kDiffNB - 1));
    bulk_load(buf0 + (uint32_t)st * (uint32_t)stage_bytes, f + pa0, pbytes, bar0 + 8 * st);
    ++pt;
    if (++pi == G) {
      pi = 0;
      ++pc;
    }
    if (++pslot == p.R) pslot = 0;
  };
  if (threadIdx.x == 0)
    while (pt < total && pt < kDiffNB) issue_next();
  int64_t t = 0;
  for (int c = 0; c < n_chunks; ++c) {
    size_t a0;
    uint32_t bytes;
    range(c, a0, bytes);
    const int64_t cw0 = wbeg + (int64_t)c * kDiffTW;
    uint32_t wq[kDiffWPW];  // (n_words < 2^32)
    uint32_t off[kDiffWPW];
    bool have[kDiffWPW], valid[kDiffWPW];
    int before[kDiffWPW], thh[kDiffWPW], thl[kDiffWPW], vr[kDiffWPW];
#pragma unroll
    for (int q = 0; q < kDiffWPW; ++q) {
      wq[q] = (uint32_t)(cw0 + q * kWarpsPerBlock + warp);
      have[q] = (int64_t)wq[q] < wend;
      const int64_t ww = have[q] ? (int64_t)wq[q] : cw0;
      const int row = (int)((uint32_t)ww / (uint32_t)p.wpr);
      const int x = (int)(ww - (int64_t)row * p.wpr) * 32 + lane;
      valid[q] = have[q] && x < p.w;
      const size_t pix = (size_t)(p.row0 + row) * p.w + (x < p.w ? x : p.w - 1);
      off[q] = (uint32_t)(pix - a0);
      before[q] = 0;
      thh[q] = INT_MAX;
      thl[q] = INT_MIN;
      vr[q] = 0;
      if (kLog) {
        if (valid[q]) {
          const float ref = p.ref[pix];
          int r = 0;
#pragma unroll
          for (int s2 = 128; s2 >= 1; s2 >>= 1)
            if (s_lut[r + s2] <= ref) r += s2;
          const int2 tt = s_th[r];
          thh[q] = tt.x;
          thl[q] = tt.y;
          vr[q] = r;
        }
      } else {
        before[q] = (int)__ldg((p.dcurr ? p.dprev : p.frames.at(p.r0 % p.R)) + pix);
      }
    }
    int fbase = 0;
    for (int i = 0; i < G; ++i, ++t) {
      const int st = (int)(t & (kDiffNB - 1));
      mbar_wait(bar0 + 8 * st, (uint32_t)((t / kDiffNB) & 1));
      const uint8_t* sb = s_raw + (size_t)st * stage_bytes;
      // the pair's bytes of this warp's words first (8 loads in flight), then
      // the rule; the staging address is one add per pair
      int val[kDiffWPW];
#pragma unroll
      for (int q = 0; q < kDiffWPW; ++q) val[q] = (int)sb[off[q]];
      const uint32_t sta = pin(st_b + (uint32_t)(i - fbase) * 8u);
#pragma unroll
      for (int q = 0; q < kDiffWPW; ++q) {
        uint2 m;
        if (kLog) {
          m = dense_rule_th(th_b, val[q], thh[q], thl[q], vr[q]);
        } else {
          const int d = val[q] - before[q];  // difference_frame, core.cpp:14-15
          m = make_uint2(__ballot_sync(kFull, d > p.c_pos && valid[q]), __ballot_sync(kFull, d < p.c_neg && valid[q]));
          before[q] = val[q];
        }
        if (lane == 0)
          asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(sta + (uint32_t)q * kStRow), "r"(m.x), "r"(m.y) : "memory");
      }
      __syncthreads();  // every warp is done with stage st
      if (threadIdx.x == 0 && pt < total) issue_next();
      if (i + 1 - fbase == 32 || i + 1 == G) {  // store the staged links' masks
        const int n = i + 1 - fbase;
        if (lane < n) {
#pragma unroll
          for (int q = 0; q < kDiffWPW; ++q) {
            if (!have[q]) continue;
            const uint2 m = s_stm[warp][q][lane];
            EVSIM_CHECK((size_t)(fbase + lane) * p.n_words + wq[q] < p.masks_cap, "diff chain mask store");
            p.masks[(size_t)(fbase + lane) * p.n_words + wq[q]] = m;
            const uint32_t cnt = __popc(m.x | m.y);
            if (cnt) atomicAdd(&s_cnt[fbase + lane], cnt);
          }
        }
        __syncwarp();
        fbase = i + 1;
      }
    }
    if (kLog) {
#pragma unroll
      for (int q = 0; q < kDiffWPW; ++q)
        if (valid[q]) p.ref[(size_t)off[q] + a0] = s_lut[vr[q]];
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < G; i += blockDim.x) {
    EVSIM_CHECK((size_t)i * p.n_blocks + b < p.counts_cap, "chain count store");
    p.counts[(size_t)i * p.n_blocks + b] = s_cnt[i];
  }
}

// bytes of one stage buffer: the rows kDiffTW words can span, 16-aligned on both ends
static int diff_stage_bytes(const ChainParams& p) {
  const int rows = (kDiffTW + p.wpr - 1) / p.wpr + 1;
  return (int)((((size_t)rows * p.w + 32) + 127) & ~(size_t)127);
}

static bool chain_diff_tma_ok(const ChainParams& p) {
  const uintptr_t base = p.dcurr ? (uintptr_t)p.dcurr : (uintptr_t)p.frames.base;
  const size_t stride = p.dcurr ? p.P : p.frames.stride;
  if ((base & 15) || (stride & 15) || (p.dprev && ((uintptr_t)p.dprev & 15))) return false;
  const size_t sm = (size_t)kDiffNB * diff_stage_bytes(p) + (size_t)p.n_pairs * 4;
  return sm <= 160 * 1024;
}

// ------------------------------------------------------------ lerp quads
// ------------------------------------------------------------ tile-staged dense chain
//
// chain_dense_kernel with the gather images staged in shared memory.  The
// global 16-byte gathers of the fp32 lerp quads bound that kernel by the L1
// data pipe (every quarter-warp request touches two or more lines).  Here a
// block owns a 2-D tile of kTileW words x kTileH rows (warp r = tile row r,
// its kTileW words one after another); for every pair of the launch the block
// reduces the exact bounds of its pixels' sample positions (prev is read
// along x - fwd*u between x and x - u, curr between x and x + u; rounding is
// monotone, so RN(x -/+ u) bound every link's position), bulk-copies that
// region of both frames' (a00, a10 - a00) rows into shared memory
// (cp.async.bulk global -> shared, one copy per row, completion on an
// mbarrier) and the samples become two conflict-free 8-byte LDS each (the
// bottom pair of a pixel is the top pair of the row below; the row pitch is a
// multiple of 128 bytes).  Same arithmetic on the same values as
// dense_fast(float4): bit-identical decisions.  A (tile, pair) whose region
// does not fit the staging rows falls back to the u8-quad gathers.  One
// count block = one tile row (words_per_block = kTileW), so the per-(link,
// block) counts are stored by the owning warp, no block-level accumulation.
constexpr int kTileW = 4;                    // words per tile row = words_per_block
constexpr int kTileH = kWarpsPerBlock;       // tile rows = warps
constexpr int kTilePitch = 144;              // float2 per staged row (128 px + flow extent <= 16)
constexpr uint32_t kTilePB = kTilePitch * 8; // bytes per staged row (9 x 128)

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// mbar_wait with a suspend-time hint: the waiting warps sleep in the barrier
// unit instead of spinning on the issue slots the other resident blocks need
__device__ __forceinline__ void mbar_wait_hint(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITH_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAITH_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity), "r"(0x989680u)
      : "memory");
}
__device__ __forceinline__ void bulk_load_tx(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

template <bool kClamp>
__device__ __forceinline__ int dense_fast_tile(const uint8_t* __restrict__ s_reg, uint32_t ba, uint32_t bb, float my,
                                               float wm, float hm, float xf, float yf, float u, float v, float4 kc,
                                               unsigned& bad, unsigned bit, uint32_t lim_a, uint32_t lim_b) {
  const f32x2 NB = pk2(kc.x, kc.y);
  f32x2 X = affine2_est(xf, NB, u), Y = affine2_est(yf, NB, v);
  if (kClamp) {
    X = pk2(fminf(fmaxf(lo2(X), 0.0f), wm), fminf(fmaxf(hi2(X), 0.0f), wm));
    Y = pk2(fminf(fmaxf(lo2(Y), 0.0f), hm), fminf(fmaxf(hi2(Y), 0.0f), hm));
  }
  const f32x2 C23 = pk2(8388608.0f, 8388608.0f);
  const f32x2 CY = pk2(my, my);
  const f32x2 TX = add2_rz(X, C23), TY = add2_rz(Y, CY);  // magic + trunc
  const f32x2 FX = sub2(X, sub2(TX, C23)), FY = sub2(Y, sub2(TY, CY));
  // byte offsets into the staged regions (ba / bb fold the magic bits and the region origins)
  const uint32_t oa = __float_as_uint(lo2(TY)) * kTilePB + (__float_as_uint(lo2(TX)) * 8u + ba);
  const uint32_t ob = __float_as_uint(hi2(TY)) * kTilePB + (__float_as_uint(hi2(TX)) * 8u + bb);
  // (checked build: both taps' rows inside the frame's staged rows; lim_a =
  // end of prev's rows = start of curr's, lim_b = end of curr's)
  EVSIM_CHECK(oa + kTilePB + 8u <= lim_a, "tile chain: prev sample inside its staged region");
  EVSIM_CHECK(ob >= lim_a && ob + kTilePB + 8u <= lim_b, "tile chain: curr sample inside its staged region");
  (void)lim_a, (void)lim_b;
  const float2 At = *reinterpret_cast<const float2*>(s_reg + oa);
  const float2 Ab = *reinterpret_cast<const float2*>(s_reg + oa + kTilePB);
  const float2 Bt = *reinterpret_cast<const float2*>(s_reg + ob);
  const float2 Bb = *reinterpret_cast<const float2*>(s_reg + ob + kTilePB);
  const float ta = __fmaf_rn(lo2(FX), At.y, At.x), ba2 = __fmaf_rn(lo2(FX), Ab.y, Ab.x);
  const float tb = __fmaf_rn(hi2(FX), Bt.y, Bt.x), bb2 = __fmaf_rn(hi2(FX), Bb.y, Bb.x);
  const float sa = __fmaf_rn(lo2(FY), __fsub_rn(ba2, ta), ta);
  const float sb = __fmaf_rn(hi2(FY), __fsub_rn(bb2, tb), tb);
  const float e = __fmaf_rn(kc.y, sa, __fmul_rn(-kc.x, sb));  // (oma_f = kc.y, alpha_f = -kc.x)
  const f32x2 T = add2_rz(add2(pk2(e, e), pk2(0.5f - 2e-4f, 0.5f + 2e-4f)), C23);
  if (__float_as_uint(lo2(T)) != __float_as_uint(hi2(T))) bad |= bit;
  return __float_as_int(hi2(T));
}

template <int kNB, bool kClamp, int kBM>
__device__ __forceinline__ unsigned dense_batch_tile(const ChainParams& p, const uint8_t* s_reg, uint32_t ba,
                                                     uint32_t bb, float my, float wm, float hm, const DenseWord& c,
                                                     int k0, int (&vals)[1][kBM], uint32_t lim_a, uint32_t lim_b) {
  unsigned bad = 0;
#pragma unroll
  for (int j = 0; j < kNB; ++j)
    vals[0][j] = dense_fast_tile<kClamp>(s_reg, ba, bb, my, wm, hm, c.xf, c.yf, c.u, c.v, p.kcp[k0 + j], bad, 1u << j,
                                        lim_a, lim_b);
  return bad;
}

template <bool kLog, int kB, int kMinB>
__global__ void __launch_bounds__(256, kMinB) chain_dense_tile_kernel(ChainParams p) {
  extern __shared__ __align__(128) uint8_t s_reg[];  // tile_cap_rows staged rows of kTilePB bytes
  __shared__ float s_lut[256];
  __shared__ int2 s_th[kLog ? 256 : 1];
  constexpr int kStage = 32 + kB;
  __shared__ uint2 s_stm[kWarpsPerBlock][kStage];
  __shared__ uint32_t s_wcnt[kWarpsPerBlock][kMaxParamK];  // the pair's events per link of this warp's row
  __shared__ int s_bnd[2][8];  // per pair parity: min (px, py, cx, cy), max (px, py, cx, cy)
  __shared__ __align__(8) uint64_t s_bar;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int L = p.d.n_links, N = p.n_interp;
  if (kLog) {
    s_lut[threadIdx.x] = p.lut[threadIdx.x];
    s_th[threadIdx.x] = make_int2(p.lthr[threadIdx.x].x, p.lthr[threadIdx.x].y);
  }
  for (int i = threadIdx.x; i < kWarpsPerBlock * kMaxParamK; i += blockDim.x) (&s_wcnt[0][0])[i] = 0;
  if (threadIdx.x < 16) (&s_bnd[0][0])[threadIdx.x] = (threadIdx.x & 4) ? INT_MIN : INT_MAX;
  const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&s_bar);
  const uint32_t reg0 = (uint32_t)__cvta_generic_to_shared(s_reg);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t w = (uint32_t)p.w;
  const float wm = (float)(p.w - 1), hm = (float)(p.h - 1);
  const float my = p.magic_y;
  const uint32_t lut_b = pin((uint32_t)__cvta_generic_to_shared(s_lut) - ((uint32_t)kVB << 2));
  const uint32_t th_b = pin((uint32_t)__cvta_generic_to_shared(s_th) - ((uint32_t)kVB << 3));
  const int kfirst = p.d.start + 1;
  const int n_int = min(L, N - p.d.start);
  // the tile: words [tx*kTileW, +kTileW) of word-grid rows [ty*kTileH, +kTileH)
  const int tiles_x = p.wpr / kTileW;
  const int ty = (int)blockIdx.x / tiles_x, tx = (int)blockIdx.x - ty * tiles_x;
  const int grid_h = (int)(p.n_words / p.wpr);
  const int trow = ty * kTileH + warp;
  const bool have = trow < grid_h;  // (the last tile row may hang over the grid)
  const int y = p.row0 + min(trow, grid_h - 1);
  const float yf = (float)y;
  const uint32_t wi0 = (uint32_t)min(trow, grid_h - 1) * (uint32_t)p.wpr + (uint32_t)(tx * kTileW);
  const uint32_t cb = (uint32_t)min(trow, grid_h - 1) * (uint32_t)tiles_x + (uint32_t)tx;
  // per-word state across the pairs (indexed in a rolled loop: local memory,
  // touched once per (word, pair))
  int st_hi[kTileW], st_lo[kTileW], st_vr[kTileW];
  float st_u[kTileW], st_v[kTileW];
#pragma unroll
  for (int q = 0; q < kTileW; ++q) {
    st_hi[q] = INT_MAX;
    st_lo[q] = INT_MIN;
    st_vr[q] = kVB;
    st_u[q] = st_v[q] = 0.0f;
    if (kLog) {
      const int x = (tx * kTileW + q) * 32 + lane;
      if (have && x < p.w) {
        const float ref = p.ref[(uint32_t)y * w + (uint32_t)x];
        int r = 0;
#pragma unroll
        for (int st = 128; st >= 1; st >>= 1)
          if (s_lut[r + st] <= ref) r += st;
        const int2 t = s_th[r];
        st_hi[q] = t.x;
        st_lo[q] = t.y;
        st_vr[q] = kVB + r;
      }
    }
  }
  int sp = p.r0 % p.R;
  uint32_t fills = 0;
  for (int i = 0; i < p.n_pairs; ++i) {
    const int sc = sp + 1 == p.R ? 0 : sp + 1;
    const uint32_t* qp = p.quads.at(sp);
    const uint32_t* qc = p.quads.at(sc);
    const uint32_t* qbp = reinterpret_cast<const uint32_t*>(reinterpret_cast<uintptr_t>(qp) - 4ull * p.qshift);
    const uint32_t* qbc = reinterpret_cast<const uint32_t*>(reinterpret_cast<uintptr_t>(qc) - 4ull * p.qshift);
    PairCtx pc{};
    pc.pu = p.g0.pu + (size_t)i * p.g0.pair_stride;
    pc.pv = p.g0.pv + (size_t)i * p.g0.pair_stride;
    // ---- the pair's flow at this row's pixels and the tile's sample bounds
    if (have) {
      int lo0 = INT_MAX, lo1 = INT_MAX, lo2b = INT_MAX, lo3 = INT_MAX;
      int hi0 = INT_MIN, hi1 = INT_MIN, hi2b = INT_MIN, hi3 = INT_MIN;
#pragma unroll
      for (int q = 0; q < kTileW; ++q) {
        const int x = min((tx * kTileW + q) * 32 + lane, p.w - 1);
        PixelCtx pxc;
        pxc.x = x;
        pxc.y = y;
        DenseProvider<false> prov;
        prov.init(p, pc, pxc);
        st_u[q] = prov.u;
        st_v[q] = prov.v;
        const float xf = (float)x;
        const float xa = fminf(fmaxf(fsub(xf, prov.u), 0.0f), wm), xb = fminf(fmaxf(fadd(xf, prov.u), 0.0f), wm);
        const float ya = fminf(fmaxf(fsub(yf, prov.v), 0.0f), hm), yb = fminf(fmaxf(fadd(yf, prov.v), 0.0f), hm);
        lo0 = min(lo0, __float2int_rz(fminf(xf, xa)));
        hi0 = max(hi0, __float2int_rz(fmaxf(xf, xa)));
        lo1 = min(lo1, __float2int_rz(fminf(yf, ya)));
        hi1 = max(hi1, __float2int_rz(fmaxf(yf, ya)));
        lo2b = min(lo2b, __float2int_rz(fminf(xf, xb)));
        hi2b = max(hi2b, __float2int_rz(fmaxf(xf, xb)));
        lo3 = min(lo3, __float2int_rz(fminf(yf, yb)));
        hi3 = max(hi3, __float2int_rz(fmaxf(yf, yb)));
      }
      lo0 = __reduce_min_sync(kFull, lo0);
      lo1 = __reduce_min_sync(kFull, lo1);
      lo2b = __reduce_min_sync(kFull, lo2b);
      lo3 = __reduce_min_sync(kFull, lo3);
      hi0 = __reduce_max_sync(kFull, hi0);
      hi1 = __reduce_max_sync(kFull, hi1);
      hi2b = __reduce_max_sync(kFull, hi2b);
      hi3 = __reduce_max_sync(kFull, hi3);
      if (lane == 0) {
        int* bn = s_bnd[i & 1];
        atomicMin(bn + 0, lo0);
        atomicMin(bn + 1, lo1);
        atomicMin(bn + 2, lo2b);
        atomicMin(bn + 3, lo3);
        atomicMax(bn + 4, hi0);
        atomicMax(bn + 5, hi1);
        atomicMax(bn + 6, hi2b);
        atomicMax(bn + 7, hi3);
      }
    }
    __syncthreads();  // bounds complete; every warp is done with the previous pair's staged rows
    const int* bn = s_bnd[i & 1];
    const int xloA = bn[0] & ~1, ncA = (bn[4] - xloA + 2) & ~1;  // even origin and count: 16-byte copies
    const int yloA = bn[1], nrA = bn[5] - yloA + 2;              // + the row below (bottom pairs)
    const int xloB = bn[2] & ~1, ncB = (bn[6] - xloB + 2) & ~1;
    const int yloB = bn[3], nrB = bn[7] - yloB + 2;
    const bool fits = ncA <= kTilePitch && ncB <= kTilePitch && nrA + nrB <= p.tile_cap_rows;
    if (threadIdx.x == 0) {  // (before this thread's mbarrier arrive / the barrier below)
#pragma unroll
      for (int k = 0; k < 8; ++k) s_bnd[(i + 1) & 1][k] = (k & 4) ? INT_MIN : INT_MAX;
    }
    if (fits) {
      if (warp == 0) {
        if (lane == 0) mbar_expect_tx(bar, (uint32_t)(nrA * ncA + nrB * ncB) * 8u);
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const float2* gA = p.quadt.at(sp);
        const float2* gB = p.quadt.at(sc);
        for (int r = lane; r < nrA + nrB; r += 32) {
          const bool isA = r < nrA;
          const int ys = min((isA ? yloA + r : yloB + r - nrA), p.h - 1);  // replicate the last row
          const float2* src = (isA ? gA : gB) + (size_t)ys * w + (isA ? xloA : xloB);
          bulk_load_tx(reg0 + (uint32_t)r * kTilePB, src, (uint32_t)(isA ? ncA : ncB) * 8u, bar);
        }
      }
      mbar_wait_hint(bar, fills & 1u);
      ++fills;
    } else {
      __syncthreads();  // (orders the s_bnd reset before the next pair's bounds)
    }
    const uint32_t BY = __float_as_uint(my);
    const uint32_t biasA = 0u - ((BY + (uint32_t)yloA) * kTilePB + (0x4B000000u + (uint32_t)xloA) * 8u);
    const uint32_t biasB =
        (uint32_t)nrA * kTilePB - ((BY + (uint32_t)yloB) * kTilePB + (0x4B000000u + (uint32_t)xloB) * 8u);
    const uint32_t lim_a = (uint32_t)nrA * kTilePB, lim_b = (uint32_t)(nrA + nrB) * kTilePB;
    // ---- the links of this row's words
    if (have) {
      const int gbase = i * L;
#pragma unroll 1
      for (int q = 0; q < kTileW; ++q) {
        DenseWord c;
        c.have = true;
        c.wi = wi0 + (uint32_t)q;
        const int x = (tx * kTileW + q) * 32 + lane;
        c.valid = x < p.w;
        c.x = x < p.w ? x : p.w - 1;
        c.y = y;
        c.pix = (uint32_t)y * w + (uint32_t)c.x;
        c.xf = (float)c.x;
        c.yf = yf;
        c.u = st_u[q];
        c.v = st_v[q];
        int thh = st_hi[q], thl = st_lo[q], vr = st_vr[q];
        float ref = 0.0f;
        int before = 0;
        // every sample x + s*u, |s| <= 1, stays in [0, w-1]: no clamp needed
        const bool safe = __all_sync(
            kFull, fabsf(c.u) <= fminf(c.xf, wm - c.xf) && fabsf(c.v) <= fminf(c.yf, hm - c.yf));
        if (!kLog)
          before = kVB + (p.d.start == 0 ? (int)p.frames.at(sp)[c.pix]
                                         : dense_exact(p.nfb, p.oma, p.alpha, qp, qc, p.w, p.h, c.xf, c.yf, c.u, c.v, 1));
        int fbase = 0;
        auto step = [&](int l, int val) {
          uint2 m;
          if constexpr (kLog) m = dense_rule_th(th_b, val, thh, thl, vr);
          else m = dense_rule<false>(p, lut_b, c, val, ref, before);
          if (lane == 0) s_stm[warp][l - fbase] = m;
        };
        auto flush = [&](int lend, bool force) {
          const int n = lend - fbase;
          if (n < 32 && !force) return;
          __syncwarp();
          for (int j = lane; j < n; j += 32) {
            const int g = gbase + fbase + j;
            const uint2 m = s_stm[warp][j];
            EVSIM_CHECK((size_t)g * p.n_words + c.wi < p.masks_cap, "tile chain mask store");
            p.masks[(size_t)g * p.n_words + c.wi] = m;
            s_wcnt[warp][fbase + j] += __popc(m.x | m.y);  // a pixel crosses one way or not at all
          }
          __syncwarp();
          fbase = lend;
        };
        for (int l0 = 0; l0 < n_int; l0 += kB) {
          const int nb = min(kB, n_int - l0);
          int vals[1][kB];
          unsigned bad;
          if (nb == kB) {
            if (fits)
              bad = safe ? dense_batch_tile<kB, false>(p, s_reg, biasA, biasB, my, wm, hm, c, kfirst + l0, vals, lim_a, lim_b)
                         : dense_batch_tile<kB, true>(p, s_reg, biasA, biasB, my, wm, hm, c, kfirst + l0, vals, lim_a, lim_b);
            else
              bad = safe ? dense_batch<1, kB, false>(p, qbp, qbc, w, my, wm, hm, &c, kfirst + l0, vals)
                         : dense_batch<1, kB, true>(p, qbp, qbc, w, my, wm, hm, &c, kfirst + l0, vals);
          } else {
            bad = 0;
            for (int j = 0; j < nb; ++j) {
              int v1[1][kB];
              unsigned b1;
              if (fits)
                b1 = safe ? dense_batch_tile<1, false>(p, s_reg, biasA, biasB, my, wm, hm, c, kfirst + l0 + j, v1, lim_a, lim_b)
                          : dense_batch_tile<1, true>(p, s_reg, biasA, biasB, my, wm, hm, c, kfirst + l0 + j, v1, lim_a, lim_b);
              else
                b1 = safe ? dense_batch<1, 1, false>(p, qbp, qbc, w, my, wm, hm, &c, kfirst + l0 + j, v1)
                          : dense_batch<1, 1, true>(p, qbp, qbc, w, my, wm, hm, &c, kfirst + l0 + j, v1);
              bad |= b1 << j;
#pragma unroll
              for (int jj = 0; jj < kB; ++jj)
                if (jj == j) vals[0][jj] = v1[0][0];
            }
          }
          if (__any_sync(kFull, bad != 0u)) {
#pragma unroll
            for (int j = 0; j < kB; ++j)
              if ((bad >> j) & 1u)
                vals[0][j] = kVB + dense_exact(p.nfb, p.oma, p.alpha, qp, qc, p.w, p.h, c.xf, c.yf, c.u, c.v,
                                               kfirst + l0 + j);
          }
          if (nb == kB) {  // (straight-line: the rule's loads stay predicated)
#pragma unroll
            for (int j = 0; j < kB; ++j) step(l0 + j, vals[0][j]);
          } else {
#pragma unroll
            for (int j = 0; j < kB; ++j) {
              if (j >= nb) break;
              step(l0 + j, vals[0][j]);
            }
          }
          flush(l0 + nb, false);
        }
        if (n_int < L) step(L - 1, kVB + (int)p.frames.at(sc)[c.pix]);  // the link into curr (include_endpoints)
        flush(L, true);
        st_hi[q] = thh;
        st_lo[q] = thl;
        st_vr[q] = vr;
      }
      // the row segment is one count block: its events per link of this pair
      for (int l = lane; l < L; l += 32) {
        EVSIM_CHECK((size_t)(gbase + l) * p.n_blocks + cb < p.counts_cap, "tile chain count store");
        p.counts[(size_t)(gbase + l) * p.n_blocks + cb] = s_wcnt[warp][l];
        s_wcnt[warp][l] = 0;
      }
      __syncwarp();
    }
    sp = sc;
  }
  if (kLog && have) {
#pragma unroll
    for (int q = 0; q < kTileW; ++q) {
      const int x = (tx * kTileW + q) * 32 + lane;
      if (x < p.w) p.ref[(uint32_t)y * w + (uint32_t)x] = s_lut[st_vr[q] - kVB];
    }
  }
}

// The dense chain's gather image of a frame: per pixel (a00 - x*dx, dx =
// a10 - a00, dy - x*dxy, dxy = (a11 - a01) - (a10 - a00)), dy = a01 - a00, in fp32 — the four taps sample_u8 reads at (x0, y0)
// (simulate.cpp:10-26, replicate clamp) with the row differences formed
// (exactly: integers).  One column per thread, kLQRows rows per block (the
// row below's taps are the next row's top taps), one 16-byte store per pixel.
constexpr int kLQRows = 8;
__device__ __forceinline__ void put_quad(float4* q, int x, float a00, float a10, float a01, float a11) {
  // (a00 - x*dx, dx, dy - x*dxy, dxy): integers, |.| <= 255 + 510 * (w - 1) < 2^24 (kLerpQuadMaxW)
  const int dx = (int)a10 - (int)a00, dy = (int)a01 - (int)a00, dxy = ((int)a11 - (int)a01) - dx;
  *q = make_float4((float)((int)a00 - x * dx), (float)dx, (float)(dy - x * dxy), (float)dxy);
}
__device__ __forceinline__ void put_quad(uint2* q, int, float a00, float a10, float a01, float a11) {
  // bf16 = the high half of the (exactly representable) fp32
  *q = make_uint2((__float_as_uint(a00) >> 16) | (__float_as_uint(a10 - a00) & 0xFFFF0000u),
                  (__float_as_uint(a01) >> 16) | (__float_as_uint(a11 - a01) & 0xFFFF0000u));
}
// tile-staged chain (chain_dense_tile_kernel): the top pair only — a pixel's
// bottom pair is the top pair of the row below (replicate-clamped)
__device__ __forceinline__ void put_quad(float2* q, int, float a00, float a10, float, float) {
  *q = make_float2(a00, a10 - a00);
}
template <class T>
__global__ void __launch_bounds__(256) lerp_quad_kernel(Ring<const uint8_t> frames, Ring<T> out, int w, int h, int R,
                                                        int slot0) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= w) return;
  const int slot = (slot0 + (int)blockIdx.z) % R;
  const uint8_t* __restrict__ f = frames.at(slot);
  T* __restrict__ q = out.at(slot);
  const int x1 = min(x + 1, w - 1);
  const int yb = blockIdx.y * kLQRows, ye = min(yb + kLQRows, h);
  float a00 = (float)__ldg(f + (size_t)yb * w + x), a10 = (float)__ldg(f + (size_t)yb * w + x1);
  for (int y = yb; y < ye; ++y) {
    const size_t r1 = (size_t)min(y + 1, h - 1) * w;
    const float a01 = (float)__ldg(f + r1 + x), a11 = (float)__ldg(f + r1 + x1);
    put_quad(q + (size_t)y * w + x, x, a00, a10, a01, a11);
    a00 = a01;
    a10 = a11;
  }
}

void launch_lerp_quads(Ring<const uint8_t> frames, Ring<float4> out, int w, int h, int R, int slot0, int n_frames,
                       cudaStream_t s) {
  if (n_frames <= 0) return;
  dim3 g((w + 255) / 256, (h + kLQRows - 1) / kLQRows, n_frames);
  lerp_quad_kernel<float4><<<g, 256, 0, s>>>(frames, out, w, h, R, slot0);
}
void launch_lerp_quads_bf16(Ring<const uint8_t> frames, Ring<uint2> out, int w, int h, int R, int slot0, int n_frames,
                            cudaStream_t s) {
  if (n_frames <= 0) return;
  dim3 g((w + 255) / 256, (h + kLQRows - 1) / kLQRows, n_frames);
  lerp_quad_kernel<uint2><<<g, 256, 0, s>>>(frames, out, w, h, R, slot0);
}

void launch_lerp_quads_f2(Ring<const uint8_t> frames, Ring<float2> out, int w, int h, int R, int slot0, int n_frames,
                          cudaStream_t s) {
  if (n_frames <= 0) return;
  dim3 g((w + 255) / 256, (h + kLQRows - 1) / kLQRows, n_frames);
  lerp_quad_kernel<float2><<<g, 256, 0, s>>>(frames, out, w, h, R, slot0);
}

// ------------------------------------------------------------ sparse chain kernel
//
// chain_kernel specialised for the sparse method (simulate.cpp:167-201): the
// intermediate frame k is prev except where a splat claimed the pixel.  A
// link whose value is prev (v0) for every lane of the word, right after a
// link that also ended in v0 for every lane, cannot emit (linear: the
// difference is 0; log: |L(v0) - ref| <= C was just established or ref =
// L(v0)) and leaves the state unchanged — such links only record empty masks.
// The first link of a pair qualifies in linear mode when it starts from v0,
// and in log mode when the pair's chain starts at prev (endpoints included:
// the previous link ended in this pair's prev, or ref = L(frame0)).
template <bool kLog, bool kMag>
__global__ void __launch_bounds__(256, 3) chain_sparse_kernel(ChainParams p) {
  // Work per word varies widely (only words near claimed pixels evaluate
  // links), so warps take two-word tasks from a device counter instead of a
  // static block partition (no block waits for its slowest warp); the
  // (link, block) counts the emit needs are global atomics on the word's
  // block, zeroed by the launch.
  constexpr int kW = 2;
  __shared__ float s_lut[256];
  const int L = p.d.n_links, N = p.n_interp;
  if (kLog) s_lut[threadIdx.x] = p.lut[threadIdx.x];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const size_t P = p.P;
  const int kfirst = p.d.start + 1;
  const int64_t n_tasks = (p.n_words + kW - 1) / kW;
  for (;;) {
    int64_t task = 0;
    if (lane == 0) task = (int64_t)atomicAdd(p.sched, 1u);
    task = __shfl_sync(kFull, task, 0);
    if (task >= n_tasks) break;
    const int64_t w0 = task * kW;
    const uint32_t blk = (uint32_t)(w0 / p.words_per_block);  // both words (words_per_block is even)
    DenseWord c[kW];
    float ref[kW];
    int before[kW];
    int thh[kW], thl[kW], vr[kW];  // kTh: the level's (hi, lo) and biased value
#pragma unroll
    for (int q = 0; q < kW; ++q) {
      const int64_t wq = w0 + q;
      c[q].have = wq < p.n_words;
      c[q].wi = (uint32_t)wq;
      const int64_t ww = c[q].have ? wq : w0;
      const int row = (int)((uint32_t)ww / (uint32_t)p.wpr);
      const int x = (int)(ww - (int64_t)row * p.wpr) * 32 + lane;
      c[q].valid = c[q].have && x < p.w;
      c[q].x = x < p.w ? x : p.w - 1;
      c[q].y = p.row0 + row;
      c[q].pix = (uint32_t)c[q].y * (uint32_t)p.w + (uint32_t)c[q].x;
      ref[q] = kLog ? p.ref[c[q].pix] : 0.0f;
      before[q] = 0;
    }
    // the per-pixel inputs of a pair (curr value, touched words) are loaded
    // one pair ahead, so their latency overlaps the previous pair's links;
    // prev of pair i+1 is curr of pair i
    int sp = p.r0 % p.R;
    int nv0[kW], nvc[kW];
    uint32_t ntw0[kW], ntw1[kW];
    auto prefetch = [&](int i, int sc_i) {
      const uint8_t* cur = p.frames.at(sc_i);
      const uint32_t* tp = p.touched + (size_t)i * ((N + 31) >> 5) * P;
#pragma unroll
      for (int q = 0; q < kW; ++q) {
        nvc[q] = cur[c[q].pix];
        ntw0[q] = (c[q].valid && N > 0) ? tp[c[q].pix] : 0u;
        ntw1[q] = (c[q].valid && N > 32) ? tp[P + c[q].pix] : 0u;
      }
    };
    {
      const uint8_t* pr = p.frames.at(sp);
#pragma unroll
      for (int q = 0; q < kW; ++q) nv0[q] = pr[c[q].pix];
      if (p.n_pairs > 0) prefetch(0, sp + 1 == p.R ? 0 : sp + 1);
    }
    for (int i = 0; i < p.n_pairs; ++i) {
      const int sc = sp + 1 == p.R ? 0 : sp + 1;
      PairCtx pc;
      pc.prev = p.frames.at(sp);
      pc.curr = p.frames.at(sc);
      pc.touched = p.touched + (size_t)i * ((N + 31) >> 5) * P;
      pc.skip = p.skip_empty && p.n_points[i] == 0;
      const uint8_t* svals = p.svals + (size_t)i * N * P;
      sp = sc;
      int v0[kW], vc[kW];
      uint32_t tw0[kW], tw1[kW], at0[kW], at1[kW];
#pragma unroll
      for (int q = 0; q < kW; ++q) {
        v0[q] = nv0[q];
        vc[q] = nvc[q];
        tw0[q] = ntw0[q];
        tw1[q] = ntw1[q];
        nv0[q] = vc[q];
      }
      if (i + 1 < p.n_pairs) prefetch(i + 1, sc + 1 == p.R ? 0 : sc + 1);
      const int gbase = i * L;
      uint2 lm[kW];
      uint32_t lwc[kW], lcnt = 0;
#pragma unroll
      for (int q = 0; q < kW; ++q) lm[q] = make_uint2(0u, 0u), lwc[q] = 0u;
      auto flush = [&](int l) {
        if ((l & 31) != 31 && l != L - 1) return;
        if (lane <= (l & 31)) {
          const int g = gbase + (l & ~31) + lane;
#pragma unroll
          for (int q = 0; q < kW; ++q) {
            if (!c[q].have) continue;
            EVSIM_CHECK((size_t)g * p.n_words + c[q].wi < p.masks_cap, "sparse chain mask store");
            p.masks[(size_t)g * p.n_words + c[q].wi] = lm[q];
            if (kMag) p.wcount[(size_t)g * p.n_words + c[q].wi] = lwc[q];
          }
          EVSIM_CHECK((size_t)g * p.n_blocks + blk < p.counts_cap, "sparse chain count");
          if (lcnt) atomicAdd(&p.counts[(size_t)g * p.n_blocks + blk], lcnt);
        }
        lcnt = 0;
      };
      if (pc.skip) {  // log mode, no endpoints, nothing selected: no events
#pragma unroll
        for (int q = 0; q < kW; ++q) lm[q] = make_uint2(0u, 0u);
        for (int l = 0; l < L; ++l) flush(l);
        continue;
      }
#pragma unroll
      for (int q = 0; q < kW; ++q) {
        at0[q] = __reduce_or_sync(kFull, tw0[q]);
        at1[q] = __reduce_or_sync(kFull, tw1[q]);
      }
      // value of interior chain frame k (1..N) at this lane; consumes the claim
      auto value = [&](int q, int k) -> int {
        const int bit = k - 1;
        bool t;
        if (bit < 32) t = (tw0[q] >> bit) & 1u;
        else if (bit < 64) t = (tw1[q] >> (bit - 32)) & 1u;
        else t = c[q].valid && ((pc.touched[(size_t)(bit >> 5) * P + c[q].pix] >> (bit & 31)) & 1u);
        return t ? (int)svals[(size_t)bit * P + c[q].pix] : v0[q];
      };
      auto any_touched = [&](int q, int k) -> bool {
        const int bit = k - 1;
        if (bit < 32) return (at0[q] >> bit) & 1u;
        if (bit < 64) return (at1[q] >> (bit - 32)) & 1u;
        return true;
      };
      // links that must be evaluated, as a bit set over l (bit l of ev64):
      // an interior link ending in k (bit k-1 of the any-touched set A) is
      // skipped when neither k nor the frame before it has a touched lane;
      // the first link also needs a v0 start (see above); curr always counts
      uint64_t ev64[kW];
      const int nint = min(L, N - p.d.start);  // links ending in an interior frame
#pragma unroll
      for (int q = 0; q < kW; ++q) {
        bool same0;
        if (p.d.start == 0) {
          before[q] = v0[q];
          same0 = true;
        } else {
          // chain starts at frame 1: its value is `before` (linear) and its
          // claim must be consumed in both modes
          before[q] = value(q, 1);
          same0 = !kLog && !any_touched(q, 1);
        }
        if (L > 64 || N > 64) {
          ev64[q] = ~0ull;
        } else {
          const uint64_t A = ((uint64_t)at1[q] << 32) | at0[q];  // bit k-1: frame k touched somewhere
          const uint64_t Al = A >> p.d.start;                     // bit l: link l's end frame touched
          uint64_t e = Al | (Al << 1) | (same0 ? 0ull : 1ull);
          e &= nint >= 64 ? ~0ull : ((1ull << nint) - 1ull);
          if (nint < L) e |= 1ull << (L - 1);  // the link into curr
          ev64[q] = e;
        }
      }
      for (int lb = 0; lb < L; lb += 32) {
        const int nl = min(32, L - lb);
        uint32_t e32[kW];
#pragma unroll
        for (int q = 0; q < kW; ++q) e32[q] = (uint32_t)(lb < 64 ? ev64[q] >> lb : ~0ull);
        if (nl < 32) {
#pragma unroll
          for (int q = 0; q < kW; ++q) e32[q] &= (1u << nl) - 1u;
        }
        uint32_t todo = e32[0];
#pragma unroll
        for (int q = 1; q < kW; ++q) todo |= e32[q];
        while (todo) {
          // up to 4 evaluated links at once: their value loads overlap
          int js[4];
          int vals[kW][4];
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            js[m] = todo ? __ffs(todo) - 1 : -1;
            todo &= todo ? todo - 1 : 0u;
          }
#pragma unroll
          for (int m = 0; m < 4; ++m) {
#pragma unroll
            for (int q = 0; q < kW; ++q) {
              const int j = js[m];
              const int k = kfirst + lb + j;
              vals[q][m] = (j >= 0 && ((e32[q] >> j) & 1u)) ? (k <= N ? value(q, k) : vc[q]) : 0;
            }
          }
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            const int j = js[m];
            if (j < 0) break;
            const int l = lb + j;
#pragma unroll
            for (int q = 0; q < kW; ++q) {
              if (!((e32[q] >> j) & 1u)) continue;
              uint32_t ev;
              const uint2 mk =
                  link_rule<kLog, kMag>(p, s_lut, gbase + l, c[q], lane, vals[q][m], ref[q], before[q], ev);
              if (lane == j) {
                lm[q] = mk;
                if (kMag) lwc[q] = ev;
                lcnt += ev;
              }
            }
          }
        }
        // skipped links: empty masks (no events, state unchanged)
#pragma unroll
        for (int q = 0; q < kW; ++q) {
          if (!((e32[q] >> lane) & 1u)) {
            lm[q] = make_uint2(0u, 0u);
            lwc[q] = 0u;
          }
        }
        flush(lb + nl - 1);
      }
      // touched planes back to zero for the next launch
#pragma unroll
      for (int q = 0; q < kW; ++q) {
        if (!c[q].valid) continue;
        if (tw0[q]) pc.touched[c[q].pix] = 0u;
        if (tw1[q]) pc.touched[P + c[q].pix] = 0u;
        for (int wdx = 2; wdx < ((N + 31) >> 5); ++wdx)
          if (pc.touched[(size_t)wdx * P + c[q].pix]) pc.touched[(size_t)wdx * P + c[q].pix] = 0u;
      }
    }
    if (kLog) {
#pragma unroll
      for (int q = 0; q < kW; ++q)
        if (c[q].valid) p.ref[c[q].pix] = ref[q];
    }
  }
}

// ------------------------------------------------------------ difference_interp kernel
//
// difference_interp_events (simulate.cpp:212-285) as links: link k = 1..N is
// the warped difference frame k — the pixels a splat claimed, each carrying
// the winning signed d1, thresholded directly (no differencing, no state);
// the optional last link thresholds d2 = curr - prev at the interval end.
// Links with no claimed pixel in the word are skipped (empty masks).  Pair 0
// of a launch emits nothing when the stream has no previous difference frame
// (simulate.cpp:334-341).
template <bool kMag>
__global__ void __launch_bounds__(256, 3) chain_diffinterp_kernel(ChainParams p) {
  constexpr int kW = 2;
  extern __shared__ uint32_t s_cnt[];  // [G]
  const int L = p.d.n_links, G = L * p.n_pairs, N = p.n_interp;
  for (int i = threadIdx.x; i < G; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  const int b = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const size_t P = p.P;
  const int nint = min(L, N);  // links into warped difference frames
  const int64_t wbeg = (int64_t)b * p.words_per_block;
  const int64_t wend = min(wbeg + p.words_per_block, p.n_words);
  for (int64_t w0 = wbeg + warp; w0 < wend; w0 += kWarpsPerBlock * kW) {
    DenseWord c[kW];
#pragma unroll
    for (int q = 0; q < kW; ++q) {
      const int64_t wq = w0 + q * kWarpsPerBlock;
      c[q].have = wq < wend;
      c[q].wi = (uint32_t)wq;
      const int64_t ww = c[q].have ? wq : w0;
      const int row = (int)((uint32_t)ww / (uint32_t)p.wpr);
      const int x = (int)(ww - (int64_t)row * p.wpr) * 32 + lane;
      c[q].valid = c[q].have && x < p.w;
      c[q].x = x < p.w ? x : p.w - 1;
      c[q].y = p.row0 + row;
      c[q].pix = (uint32_t)c[q].y * (uint32_t)p.w + (uint32_t)c[q].x;
    }
    int sp = p.r0 % p.R;
    for (int i = 0; i < p.n_pairs; ++i) {
      const int sc = sp + 1 == p.R ? 0 : sp + 1;
      const uint8_t* prev = p.frames.at(sp);
      const uint8_t* curr = p.frames.at(sc);
      const uint32_t* touched = p.touched + (size_t)i * ((N + 31) >> 5) * P;
      const int16_t* dvals = p.dvals + (size_t)i * N * P;
      sp = sc;
      const int gbase = i * L;
      const bool skip = p.skip_first && i == 0;
      uint2 lm[kW];
      uint32_t lwc[kW], lcnt = 0;
#pragma unroll
      for (int q = 0; q < kW; ++q) lm[q] = make_uint2(0u, 0u), lwc[q] = 0u;
      auto flush = [&](int l) {
        if ((l & 31) != 31 && l != L - 1) return;
        if (lane <= (l & 31)) {
          const int g = gbase + (l & ~31) + lane;
#pragma unroll
          for (int q = 0; q < kW; ++q) {
            if (!c[q].have) continue;
            EVSIM_CHECK((size_t)g * p.n_words + c[q].wi < p.masks_cap, "sparse chain mask store");
            p.masks[(size_t)g * p.n_words + c[q].wi] = lm[q];
            if (kMag) p.wcount[(size_t)g * p.n_words + c[q].wi] = lwc[q];
          }
          if (lcnt) atomicAdd(&s_cnt[g], lcnt);
        }
        lcnt = 0;
      };
      uint32_t tw0[kW], tw1[kW];
      uint64_t ev64[kW];
#pragma unroll
      for (int q = 0; q < kW; ++q) {
        tw0[q] = (c[q].valid && N > 0 && !skip) ? touched[c[q].pix] : 0u;
        tw1[q] = (c[q].valid && N > 32 && !skip) ? touched[P + c[q].pix] : 0u;
        const uint64_t A = ((uint64_t)__reduce_or_sync(kFull, tw1[q]) << 32) | __reduce_or_sync(kFull, tw0[q]);
        uint64_t e = (N > 64 || L > 64) ? ~0ull : A & (nint >= 64 ? ~0ull : ((1ull << nint) - 1ull));
        if (nint < L && L <= 64) e |= 1ull << (L - 1);  // the d2 link
        ev64[q] = skip ? 0ull : e;
      }
      auto value = [&](int q, int k) -> int {  // signed value of link k at this lane
        if (k > N) return (int)curr[c[q].pix] - (int)prev[c[q].pix];
        const int bit = k - 1;
        bool t;
        if (bit < 32) t = (tw0[q] >> bit) & 1u;
        else if (bit < 64) t = (tw1[q] >> (bit - 32)) & 1u;
        else t = c[q].valid && ((touched[(size_t)(bit >> 5) * P + c[q].pix] >> (bit & 31)) & 1u);
        return t ? (int)dvals[(size_t)bit * P + c[q].pix] : 0;
      };
      for (int lb = 0; lb < L; lb += 32) {
        const int nl = min(32, L - lb);
        uint32_t e32[kW];
#pragma unroll
        for (int q = 0; q < kW; ++q) {
          e32[q] = (uint32_t)(lb < 64 ? ev64[q] >> lb : (skip ? 0ull : ~0ull));
          if (nl < 32) e32[q] &= (1u << nl) - 1u;
        }
        uint32_t todo = e32[0];
#pragma unroll
        for (int q = 1; q < kW; ++q) todo |= e32[q];
        while (todo) {
          int js[4];
          int vals[kW][4];
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            js[m] = todo ? __ffs(todo) - 1 : -1;
            todo &= todo ? todo - 1 : 0u;
          }
#pragma unroll
          for (int m = 0; m < 4; ++m)
#pragma unroll
            for (int q = 0; q < kW; ++q)
              vals[q][m] = (js[m] >= 0 && ((e32[q] >> js[m]) & 1u)) ? value(q, lb + js[m] + 1) : 0;
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            const int j = js[m];
            if (j < 0) break;
            const int l = lb + j;
#pragma unroll
            for (int q = 0; q < kW; ++q) {
              if (!((e32[q] >> j) & 1u)) continue;
              uint32_t ev;
              float unused_ref = 0.0f;
              int zero = 0;  // the value is the difference itself (threshold_events_into)
              const uint2 mk = link_rule<false, kMag>(p, nullptr, gbase + l, c[q], lane, vals[q][m], unused_ref,
                                                      zero, ev);
              if (lane == j) {
                lm[q] = mk;
                if (kMag) lwc[q] = ev;
                lcnt += ev;
              }
            }
          }
        }
#pragma unroll
        for (int q = 0; q < kW; ++q) {
          if (!((e32[q] >> lane) & 1u)) {
            lm[q] = make_uint2(0u, 0u);
            lwc[q] = 0u;
          }
        }
        flush(lb + nl - 1);
      }
      // touched planes back to zero for the next launch
#pragma unroll
      for (int q = 0; q < kW; ++q) {
        if (!c[q].valid || skip) continue;
        uint32_t* tp = const_cast<uint32_t*>(touched);
        if (tw0[q]) tp[c[q].pix] = 0u;
        if (tw1[q]) tp[P + c[q].pix] = 0u;
        for (int wdx = 2; wdx < ((N + 31) >> 5); ++wdx)
          if (tp[(size_t)wdx * P + c[q].pix]) tp[(size_t)wdx * P + c[q].pix] = 0u;
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < G; i += blockDim.x) {
    EVSIM_CHECK((size_t)i * p.n_blocks + b < p.counts_cap, "chain count store");
    p.counts[(size_t)i * p.n_blocks + b] = s_cnt[i];
  }
}

// ------------------------------------------------------------ offsets
// One warp per link row: exclusive prefix of the row's per-block counts and
// the row total.  Chunks of 32 blocks with a running carry.
__global__ void __launch_bounds__(256) offsets_kernel(OffsetParams p) {
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  if (row >= p.n_rows) return;
  const uint32_t* src = p.counts + (size_t)row * p.n_blocks;
  int64_t* dst = p.prefix + (size_t)row * p.n_blocks;
  int64_t carry = 0;
  for (int b0 = 0; b0 < p.n_blocks; b0 += 32) {
    const int b = b0 + lane;
    const int64_t c = b < p.n_blocks ? (int64_t)src[b] : 0;
    int64_t x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (b < p.n_blocks) dst[b] = carry + x - c;
    carry += __shfl_sync(kFull, x, 31);
  }
  if (lane == 0) p.link_total[row] = carry;
}

// Few link rows (large frames, few pairs per launch: c5 has 33 rows of ~1.2k
// blocks): one block per row, each thread a contiguous run of the row's
// counts, one block scan — instead of one warp walking the row 32 at a time.
__global__ void __launch_bounds__(256) offsets_row_kernel(OffsetParams p) {
  __shared__ int64_t s_warp[32];
  const int row = blockIdx.x;
  const uint32_t* src = p.counts + (size_t)row * p.n_blocks;
  int64_t* dst = p.prefix + (size_t)row * p.n_blocks;
  const int per = (p.n_blocks + blockDim.x - 1) / blockDim.x;
  const int b0 = min((int)threadIdx.x * per, p.n_blocks), b1 = min(b0 + per, p.n_blocks);
  int64_t sum = 0;
  for (int b = b0; b < b1; ++b) sum += src[b];
  int64_t tot;
  int64_t run = block_exclusive_scan(sum, s_warp, tot);
  for (int b = b0; b < b1; ++b) {
    const uint32_t c = src[b];
    dst[b] = run;
    run += c;
  }
  if (threadIdx.x == 0) p.link_total[row] = tot;
}

// Segment bases: exclusive scan of the segment totals (one block); also the
// host-visible segment table seg_out.
__global__ void __launch_bounds__(1024) segbase_kernel(EmitParams p, int64_t* segbase) {
  __shared__ int64_t s_warp[32];
  const int S = *p.seg.n_segs;
  const int lo = p.seg_hi ? p.seg_lo : 0, hi = p.seg_hi ? p.seg_hi : S;  // (a sub-batch's segments)
  const int64_t b0 = *p.base;  // events of earlier launches of the same call
  __syncthreads();
  int64_t carry = b0;
  for (int s0 = lo; s0 < hi; s0 += blockDim.x) {
    const int s = s0 + threadIdx.x;
    int64_t tot = 0;
    if (s < hi) {
      const int k0 = p.seg.seg_first[s], nk = p.seg.seg_nlinks[s];
      for (int k = k0; k < k0 + nk; ++k) tot += p.link_total[k];
    }
    int64_t chunk;
    const int64_t excl = block_exclusive_scan(tot, s_warp, chunk);
    if (s < hi) {
      segbase[s] = carry + excl;
      p.seg_out[1 + s] = p.seg.seg_t[s];
      p.seg_out[1 + S + s] = carry + excl;
    }
    carry += chunk;
  }
  if (threadIdx.x == 0) {
    p.seg_out[0] = S;
    p.seg_out[1 + 2 * S] = carry;
    *p.base = carry;
  }
}

// Predicated global store without a branch (the dense-word expansion's
// per-lane "has an event" condition).
__device__ __forceinline__ void st_global_if(uint32_t* ptr, uint32_t v, uint32_t cond) {
  asm volatile("{.reg .pred q; setp.ne.u32 q, %2, 0; @q st.global.u32 [%0], %1;}" ::"l"(ptr), "r"(v), "r"(cond)
               : "memory");
}

// ------------------------------------------------------------ emit kernel
//
// Writes every event once, in the reference's order (t, y, x, p).  The
// block's (segment, word) items are scanned in ONE flattened pass (chunks of
// 256), and the 8 warps expand the items round-robin with lanes = pixels:
// lane l's event lands at base + offset + popc(mask & lanemask_lt) — a
// warp-ballot compaction.  Segments with several links (equal timestamps,
// finalize's stable_sort at simulate.cpp:36-40) and magnitude mode take the
// per-lane count path: per pixel all negative events precede the positive.
__global__ void __launch_bounds__(256) emit_kernel(EmitParams p, const int64_t* __restrict__ segbase) {
  extern __shared__ int64_t s_off0[];  // [S] output offset of segment s in this block minus its flat offset
  int* s_list = reinterpret_cast<int*>(s_off0 + p.n_links);  // segments with events in this block
  __shared__ int s_warp[kWarpsPerBlock];
  __shared__ int s_item[256];
  __shared__ int64_t s_dst[256];
  __shared__ int s_nwork;
  __shared__ uint4 s_wd[kWarpsPerBlock][32];      // dense-word expansion: (all, pos, x|row<<16, -)
  __shared__ uint32_t* s_wptr[kWarpsPerBlock][32];  // and the word's first output record
  const int b = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int S = *p.seg.n_segs;
  if (p.seg_out[1 + 2 * S] > p.capacity) return;  // host grows the buffer and re-emits
  const int64_t wbeg = (int64_t)b * p.words_per_block;
  const int nw = (int)(min(wbeg + p.words_per_block, p.n_words) - wbeg);
  // segment s of this block starts at segbase[s] + sum over its links of the
  // events in earlier blocks; segments without events in this block are
  // dropped from the item list (their masks are never read)
  int n_nz = 0;
  const int slo = p.seg_hi ? p.seg_lo : 0, shi = p.seg_hi ? p.seg_hi : S;  // (a sub-batch's segments)
  for (int s0 = slo; s0 < shi; s0 += blockDim.x) {
    const int s = s0 + threadIdx.x;
    int nz = 0;
    if (s < shi) {
      const int k0 = p.seg.seg_first[s], nk = p.seg.seg_nlinks[s];
      int64_t o = segbase[s];
      uint32_t cnt = 0;
      for (int k = k0; k < k0 + nk; ++k) {
        o += p.prefix[(size_t)k * p.n_blocks + b];
        cnt += p.counts[(size_t)k * p.n_blocks + b];
      }
      s_off0[s] = o;
      nz = cnt != 0u;
    }
    int tot;
    const int pos = block_exclusive_scan(nz, s_warp, tot);
    if (nz) s_list[n_nz + pos] = s;
    n_nz += tot;
  }
  __syncthreads();
  const int n_items = n_nz * nw;
  int64_t carry = 0;
  for (int c0 = 0; c0 < n_items; c0 += blockDim.x) {
    const int it = c0 + threadIdx.x;
    const bool valid = it < n_items;
    const int si = valid ? it / nw : 0;
    const int s = valid ? s_list[si] : 0;
    const int j = valid ? it - si * nw : 0;
    uint32_t pos = 0, all = 0;
    int cnt = 0;
    bool fast = false;
    if (valid) {
      const int k0 = p.seg.seg_first[s], nk = p.seg.seg_nlinks[s];
      const int64_t wi = wbeg + j;
      fast = !p.magnitude && nk == 1;
      if (fast) {
        const uint2 m = p.masks[(size_t)k0 * p.n_words + wi];
        pos = m.x;
        all = m.x | m.y;
        cnt = __popc(all);
      } else {
        for (int k = k0; k < k0 + nk; ++k) {
          if (p.magnitude) {
            cnt += (int)p.wcount[(size_t)k * p.n_words + wi];
          } else {
            const uint2 m = p.masks[(size_t)k * p.n_words + wi];
            cnt += __popc(m.x | m.y);
          }
        }
      }
    }
    int chunk_total;
    const int excl = block_exclusive_scan(cnt, s_warp, chunk_total);
    // rebase at the segment's first item, also in a chunk without events
    // (the next chunk's scan barriers publish it)
    if (valid && j == 0) s_off0[s] -= carry + excl;
    if (chunk_total == 0) continue;  // uniform
    if (threadIdx.x == 0) s_nwork = 0;
    __syncthreads();
    // segment start in this block + this block's earlier words of the segment
    // (flattened offset relative to the segment's first item)
    const int64_t dst = valid ? s_off0[s] + carry + excl : 0;
    // ---- single-link words: warp-level load-balanced expansion.  The warp's
    // 32 words hold T events; output slot q (q = lane, lane+32, ...) belongs to
    // the word whose scan interval contains q (binary search over the warp's
    // inclusive scan) and to that word's (q - start)-th set bit (__fns).
    // Consecutive slots of one segment are consecutive addresses, so each
    // store instruction writes up to 32 adjacent events.
    {
      const int c = fast ? cnt : 0;
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
      }
      const int T = __shfl_sync(kFull, incl, 31);
      const int excl = incl - c;
      const uint32_t wi = (uint32_t)(wbeg + j);
      const int lrow = (int)p.wdiv.div(wi);
      const int x0 = (int)(wi - (uint32_t)lrow * (uint32_t)p.wpr) * 32;
      // per word: output address of its slot 0 relative to the warp's slots,
      // and its (x0, row) in one word (x < 2^16, row < 2^15)
      const long long base = (long long)dst - excl;
      const uint32_t xr = (uint32_t)x0 | ((uint32_t)(p.row0 + lrow) << 16);
      const unsigned nzw = __ballot_sync(kFull, c > 0);
      const int nnz = __popc(nzw);
      if (T >= 5 * nnz && nnz >= 16) {
        // dense words (>= 5 events each on average, most words non-empty):
        // word by word with lanes = its pixels — rank = popc below the lane,
        // one coalesced run per word, no per-event search; four independent
        // words per step
        s_wd[warp][lane] = make_uint4(all, all & ~pos, xr, 0u);  // (events, negative events, x0 | row << 16)
        s_wptr[warp][lane] = p.out + dst;
        __syncwarp();
        const uint32_t bit = 1u << lane, below = bit - 1u;
#pragma unroll 1
        for (int k0 = 0; k0 < 32; k0 += 4) {
          uint4 wd[4];
          uint32_t* wp[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            wd[k] = s_wd[warp][k0 + k];
            wp[k] = s_wptr[warp][k0 + k];
          }
#pragma unroll
          for (int k = 0; k < 4; ++k)  // x0 is a multiple of 32: x0 + lane = x0 | lane
            st_global_if(wp[k] + __popc(wd[k].x & below), wd[k].z | (uint32_t)lane | ((wd[k].y >> lane) << 31),
                         wd[k].x & bit);
        }
        __syncwarp();
      } else
      for (int q = lane; q - lane < T; q += 32) {
        // first lane l with incl[l] > q
        int lo = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
          const int probe = __shfl_sync(kFull, incl, lo + step - 1);
          if (probe <= q) lo += step;
        }
        const int src = lo < 31 ? lo : 31;
        const int sexcl = __shfl_sync(kFull, excl, src);
        const uint32_t m = __shfl_sync(kFull, all, src);
        const uint32_t pm = __shfl_sync(kFull, pos, src);
        const long long sb = __shfl_sync(kFull, base, src);
        const uint32_t sxr = __shfl_sync(kFull, xr, src);
        if (q < T) {
          const int bit = nth_set_bit(m, q - sexcl);
          p.out[sb + q] = (sxr + (uint32_t)bit) | (((pm >> bit) & 1u) ? 0u : 0x80000000u);
        }
      }
    }
    // ---- multi-link (equal timestamps) and magnitude words: per-lane counts
    if (valid && !fast && cnt > 0) {
      const int slot = atomicAdd(&s_nwork, 1);
      s_item[slot] = it;
      s_dst[slot] = dst;
    }
    __syncthreads();
    const int nwork = s_nwork;
    for (int jj = warp; jj < nwork; jj += kWarpsPerBlock) {
      const int item = s_item[jj];
      const int sij = item / nw;
      const int sj = s_list[sij];
      const uint32_t wij = (uint32_t)(wbeg + (item - sij * nw));
      const int lrow = (int)p.wdiv.div(wij);
      const int x = (int)(wij - (uint32_t)lrow * (uint32_t)p.wpr) * 32 + lane;
      const int row = p.row0 + lrow;
      const int k0 = p.seg.seg_first[sj], nk = p.seg.seg_nlinks[sj];
      int nneg = 0, npos = 0;
      for (int k = k0; k < k0 + nk; ++k) {
        const uint2 m = p.masks[(size_t)k * p.n_words + wij];
        const int mult = p.magnitude ? (int)p.mcount[(size_t)k * p.n_words * 32 + (size_t)wij * 32 + lane] : 1;
        if ((m.x >> lane) & 1u) npos += mult;
        if ((m.y >> lane) & 1u) nneg += mult;
      }
      int incl = nneg + npos;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
      }
      int64_t d = s_dst[jj] + incl - (nneg + npos);
      for (int q = 0; q < nneg; ++q) p.out[d++] = pack_event(x, row, true);
      for (int q = 0; q < npos; ++q) p.out[d++] = pack_event(x, row, false);
    }
    __syncthreads();
    carry += chunk_total;
  }
}

// ------------------------------------------------------------ emit (single-link segments)
//
// The common case — every link its own timestamp, one event per crossing:
// segment g is link g, its events are the set bits of its masks in word
// order (threshold_events_into's (y, x) scan, src/core.cpp:21-46).  One CTA
// per (tile of chain blocks, link): a thread per 32-pixel word, a block scan
// of the words' popcounts gives each word's slot, the thread expands its set
// bits into shared memory (highest pixel first with FLO, written back to
// front), and one thread streams the tile's contiguous run to
// global memory with a TMA bulk copy (cp.async.bulk smem -> global); the
// staging buffer is offset so it has the destination's alignment mod 16 B,
// the < 16-byte head and tail go out as plain stores.  The tile starts at
// segbase[g] + the chain's per-(link, block) exclusive prefix.
__global__ void __launch_bounds__(256) emit_single_kernel(EmitParams p, const int64_t* __restrict__ segbase,
                                                          int blocks_per_tile, int g0, int g1, int links_per_block) {
  __shared__ __align__(16) uint32_t s_ev[256 * 32 + 4];
  __shared__ int s_tot[2][kWarpsPerBlock];  // the warps' event totals, double-buffered by link parity
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ga = g0 + (int)blockIdx.y * links_per_block, gb = min(ga + links_per_block, g1);
  const int b0 = blockIdx.x * blocks_per_tile;
  const int64_t w0 = (int64_t)b0 * p.words_per_block;
  const int64_t w1 = min(w0 + (int64_t)blocks_per_tile * p.words_per_block, p.n_words);
  const int64_t w = w0 + threadIdx.x;
  const bool in = w < w1;
  // a block emits one tile of words for links [ga, gb): the tile geometry,
  // the capacity check and the word's (x, y) once; each link's masks and
  // output offset are loaded one link ahead
  const int S = *p.seg.n_segs;
  const uint32_t row = p.wdiv.div((uint32_t)(in ? w : w0));
  const uint32_t xy = ((uint32_t)(in ? w : w0) - row * (uint32_t)p.wpr) * 32u | ((uint32_t)(p.row0 + (int)row) << 16);
  uint2 m_next = in ? p.masks[(size_t)ga * p.n_words + w] : make_uint2(0u, 0u);
  int64_t off_next = segbase[ga] + p.prefix[(size_t)ga * p.n_blocks + b0];
  if (p.seg_out[1 + 2 * S] > p.capacity) return;  // host grows the buffer and re-emits
  for (int g = ga; g < gb; ++g) {
    const uint2 m = m_next;
    const int64_t tile_off = off_next;
    if (g + 1 < gb) {
      m_next = in ? p.masks[(size_t)(g + 1) * p.n_words + w] : make_uint2(0u, 0u);
      off_next = segbase[g + 1] + p.prefix[(size_t)(g + 1) * p.n_blocks + b0];
    }
    const uint32_t all = m.x | m.y, neg = m.y;
    // block scan of the words' event counts with ONE barrier: a warp scan,
    // the 8 warp totals through shared memory (double-buffered by link
    // parity, so the next link's totals need no second barrier), and two
    // REDUX sums for the tile's total and the warps before this one.  The
    // barrier also orders the previous link's staged reads (head / tail
    // lanes, and the bulk copy thread 0 waited for) before this link's writes.
    const int nev = __popc(all);
    int incl = nev;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += y;
    }
    int* tot = s_tot[(g - ga) & 1];
    if (lane == 31) tot[warp] = incl;
    __syncthreads();
    const int wt = lane < kWarpsPerBlock ? tot[lane] : 0;
    const int total = __reduce_add_sync(kFull, wt);
    if (total == 0) continue;  // uniform
    const int excl = __reduce_add_sync(kFull, lane < warp ? wt : 0) + incl - nev;
    uint32_t* dst = p.out + tile_off;
    EVSIM_CHECK(tile_off >= 0 && tile_off + total <= p.capacity, "emit tile within the event buffer");
    EVSIM_CHECK(total <= 256 * 32, "emit staging size");
    const int shift = (int)(((uintptr_t)dst >> 2) & 3u);  // dst alignment mod 16 B, in events
    if (all) {
      // descending pixels (FLO = the highest set bit), written back to front;
      // n1 = neg rotated right by 1, so rotr(n1, b) holds pixel b's polarity
      // at bit 31
      const uint32_t n1 = __funnelshift_r(neg, neg, 1);
      uint32_t mm = all;
      uint32_t* o = s_ev + shift + excl + __popc(all) - 1;
      do {
        uint32_t bit;
        asm("bfind.u32 %0, %1;" : "=r"(bit) : "r"(mm));  // FLO: the highest set bit
        mm ^= 1u << bit;
        *o-- = (xy + bit) | (__funnelshift_r(n1, n1, bit) & 0x80000000u);
      } while (mm);
    }
    __syncthreads();
    const int head = min(total, (4 - shift) & 3);
    const int nbody = (total - head) & ~3;
    if ((int)threadIdx.x < head) dst[threadIdx.x] = s_ev[shift + threadIdx.x];
    const int t0 = head + nbody;
    if ((int)threadIdx.x >= 32 && (int)threadIdx.x - 32 < total - t0)
      dst[t0 + threadIdx.x - 32] = s_ev[shift + t0 + threadIdx.x - 32];
    if (threadIdx.x == 0 && nbody > 0) {
      const uint32_t src = (uint32_t)__cvta_generic_to_shared(s_ev + shift + head);
      asm volatile("fence.proxy.async.shared::cta;\n"
                   "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n"
                   "cp.async.bulk.commit_group;\n"
                   "cp.async.bulk.wait_group.read 0;\n" ::"l"(dst + head), "r"(src), "r"(nbody * 4)
                   : "memory");
    }
    // (no barrier here: the next link's scan barrier comes before its staging writes)
  }
}

// ------------------------------------------------------------ unpack
// Packed record -> evsim::Event layout (24 B: x@0 y@2 t@8 p@16).
__global__ void unpack_kernel(const uint32_t* __restrict__ packed, const int64_t* __restrict__ seg_out, int64_t n,
                              unsigned long long* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int S = (int)seg_out[0];
  const int64_t* st = seg_out + 1;
  const int64_t* so = seg_out + 1 + S;
  int lo = 0, hi = S - 1;  // last segment with offset <= i
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (so[mid] <= i) lo = mid;
    else hi = mid - 1;
  }
  const uint32_t e = packed[i];
  out[3 * i + 0] = (unsigned long long)(e & 0x7FFFFFFFu);
  out[3 * i + 1] = (unsigned long long)st[lo];
  out[3 * i + 2] = (e >> 31) ? 0xFFull : 0x01ull;
}

// ------------------------------------------------------------ interpolate_frames
// Single pair (ring slots r0, r0+1), caller-supplied flow field.
__global__ void interp_frames_kernel(ChainParams p, uint8_t* __restrict__ out) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  if (x >= p.w) return;
  PixelCtx c;
  c.valid = true;
  c.x = x;
  c.y = y;
  c.pix = (size_t)y * p.w + x;
  c.xf = (float)x;
  c.yf = (float)y;
  const PairCtx pc = pair_ctx(p, 0);
  DenseProvider<true> prov;
  prov.init(p, pc, c);
  const size_t P = (size_t)p.w * p.h;
  for (int k = 1; k <= p.n_interp; ++k) out[(size_t)(k - 1) * P + c.pix] = (uint8_t)prov.interp(p, pc, c, k);
}

// ------------------------------------------------------------ sparse selection
// |curr - prev| > sel in scan order (simulate.cpp:149-159); log mode:
// |L(curr) - L(prev)| > sel_log.  blockIdx.y = pair.
__global__ void __launch_bounds__(256) select_mask_kernel(SelectParams p) {
  __shared__ uint32_t s_cnt;
  __shared__ float s_lut[256];
  if (threadIdx.x == 0) s_cnt = 0;
  if (p.log_mode) s_lut[threadIdx.x] = p.lut[threadIdx.x];
  __syncthreads();
  const int z = blockIdx.y;
  // sparse: (prev, curr) of the pair; difference_interp: (f[r0+z-1], f[r0+z]) = d1
  const int zoff = p.diff_mode ? -1 : 0;
  auto wrap = [&](int s) {  // s in [0, 3R): s mod R without a division
    if (s >= p.R) s -= p.R;
    if (s >= p.R) s -= p.R;
    return s;
  };
  const uint8_t* prev = p.frames.at(wrap(p.r0 % p.R + z + zoff + p.R));
  const uint8_t* curr = p.frames.at(wrap(p.r0 % p.R + z + 1 + zoff));
  const bool none = p.diff_mode && p.skip_first && z == 0;
  uint32_t* masks = p.masks + (size_t)z * p.n_words;
  const int b = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t wbeg = (int64_t)b * p.words_per_block;
  const int64_t wend = min(wbeg + p.words_per_block, p.n_words);
  // (row, word column) of the warp's first word, then advanced incrementally
  int row = (int)((uint32_t)(wbeg + warp) / (uint32_t)p.wpr);
  int col = (int)(wbeg + warp - (int64_t)row * p.wpr);
  for (int64_t wi = wbeg + warp; wi < wend; wi += kWarpsPerBlock) {
    const int x = col * 32 + lane, wrow = row;
    col += kWarpsPerBlock;
    while (col >= p.wpr) col -= p.wpr, ++row;  // (rows of fewer than 8 words wrap more than once)
    bool take = false;
    if (x < p.w && !none) {
      const size_t i = (size_t)wrow * p.w + x;
      const int a = prev[i], c = curr[i];
      if (p.diff_mode) {
        const int d = c - a;
        take = d > p.c_pos || d < p.c_neg;
      } else if (p.log_mode) {
        take = fabsf(fsub(s_lut[c], s_lut[a])) > p.sel_log;
      } else {
        take = abs(c - a) > p.sel;
      }
    }
    const unsigned m = __ballot_sync(kFull, take);
    if (lane == 0) {
      masks[wi] = m;
      if (m) atomicAdd(&s_cnt, (uint32_t)__popc(m));
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) p.counts[(size_t)z * p.n_blocks + b] = s_cnt;
}

// Compact the selection into pixel indices (scan order); block 0 of each
// pair publishes M.
__global__ void __launch_bounds__(256) select_emit_kernel(SelectParams p) {
  __shared__ int s_warp[kWarpsPerBlock];

  __shared__ uint32_t s_m[256];
  __shared__ int s_off[256];
  const int z = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // this block's offset and the pair's total (offsets_kernel over the counts)
  const int64_t p_all = p.prefix[(size_t)z * p.n_blocks + blockIdx.x];
  if (blockIdx.x == 0 && threadIdx.x == 0) p.n_points[z] = (int)p.total[z];
  const uint32_t* masks = p.masks + (size_t)z * p.n_words;
  uint32_t* points = p.points + (size_t)z * p.P;
  const int64_t wbeg = (int64_t)blockIdx.x * p.words_per_block;
  const int64_t wend = min(wbeg + p.words_per_block, p.n_words);
  int64_t base = p_all;
  for (int64_t cbeg = wbeg; cbeg < wend; cbeg += blockDim.x) {
    const int64_t wi = cbeg + threadIdx.x;
    const uint32_t m = wi < wend ? masks[wi] : 0u;
    int tot32;
    const int off = block_exclusive_scan((int)__popc(m), s_warp, tot32);
    if (tot32 > 0) {
      s_m[threadIdx.x] = m;
      s_off[threadIdx.x] = off;
      __syncthreads();
      const int nvalid = (int)(wend - cbeg < 256 ? wend - cbeg : 256);
      for (int j = warp; j < nvalid; j += kWarpsPerBlock) {
        const uint32_t mj = s_m[j];
        if (!mj) continue;
        if ((mj >> lane) & 1u) {
          const uint32_t wij = (uint32_t)(cbeg + j);
          const int row = (int)(wij / (uint32_t)p.wpr);
          const int x = (int)(wij - (uint32_t)row * (uint32_t)p.wpr) * 32 + lane;
          points[base + s_off[j] + __popc(mj & lanemask_lt())] = (uint32_t)row * (uint32_t)p.w + (uint32_t)x;
        }
      }
      __syncthreads();
    }
    base += tot32;
  }
}

// ------------------------------------------------------------ sparse splat
// One thread per (point, k): simulate.cpp:175-199.  The claim rule (first
// claim, replaced only by a strictly larger change) selects, per target pixel,
// the point with the largest change and, among equals, the smallest scan
// index j: an atomicMax on (change << 24) | (2^24 - 1 - j)  (M < 2^24).
// Target slot, value and claim key of splat item (j, k); false when the
// point is lost or the target falls outside the frame.
// difference_interp (diff_mode): the value is the point's signed d1 =
// prev[src] - pprev[src] and the claim goes to the largest |d1|
// (simulate.cpp:248-255), ties to the smallest j as in the sparse rule.
__device__ __forceinline__ bool splat_item(const SplatParams& p, const uint8_t* prev, const uint8_t* pprev,
                                           const uint32_t* points, const float2* disp, const uint8_t* status,
                                           int64_t j, int k, size_t& slot, int& value, uint32_t& key) {
  if (!status[j]) return false;
  const uint32_t src = points[j];
  const int px = (int)(src % (uint32_t)p.w), py = (int)(src / (uint32_t)p.w);
  const float alpha = __fdiv_rn((float)k, (float)(p.n_interp + 1));
  const float2 d = disp[j];
  const int tx = lroundf_ref(fadd((float)px, fmul(alpha, d.x)));
  const int ty = lroundf_ref(fadd((float)py, fmul(alpha, d.y)));
  if (tx < 0 || tx >= p.w || ty < 0 || ty >= p.h) return false;
  const size_t idx = (size_t)ty * p.w + tx;
  int change;
  if (p.diff_mode) {
    value = (int)prev[src] - (int)pprev[src];
    change = abs(value);
  } else {
    value = prev[src];
    change = abs(value - (int)prev[idx]);
  }
  key = ((uint32_t)change << 24) | (0xFFFFFFu - (uint32_t)j);
  slot = (size_t)(k - 1) * p.P + idx;
  return true;
}

__global__ void splat_kernel(SplatParams p) {
  const int z = blockIdx.y;
  const int64_t M = p.n_points[z];
  const int N = p.n_interp;
  const int64_t total = M * N;
  const size_t P = p.P;
  const uint8_t* prev = p.frames.at((p.r0 + z) % p.R);
  const uint8_t* pprev = p.frames.at((p.r0 + z - 1 + p.R) % p.R);
  const uint32_t* points = p.points + (size_t)z * P;
  const float2* disp = p.disp + (size_t)z * P;
  const uint8_t* status = p.status + (size_t)z * P;
  uint32_t* claims = p.claims + (size_t)z * N * P;
  uint32_t* touched = p.touched + (size_t)z * ((N + 31) / 32) * P;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / N;
    const int k = (int)(e - j * N) + 1;
    size_t slot;
    int value;
    uint32_t key;
    if (!splat_item(p, prev, pprev, points, disp, status, j, k, slot, value, key)) continue;
    atomicMax(&claims[slot], key);
    const size_t idx = slot - (size_t)(k - 1) * P;
    atomicOr(&touched[(size_t)((k - 1) >> 5) * P + idx], 1u << ((k - 1) & 31));
  }
}

// After the claims settle: the winner of every claimed slot stores its value
// (the intermediate frame's pixel, simulate.cpp:195-197) in the u8 value plane
// and zeroes the claim, so the chain reads one byte per touched pixel and the
// claim planes are clean for the next launch.  Keys are unique per point, so
// only the winner matches.
__global__ void resolve_kernel(SplatParams p) {
  const int z = blockIdx.y;
  const int64_t M = p.n_points[z];
  const int N = p.n_interp;
  const int64_t total = M * N;
  const size_t P = p.P;
  const uint8_t* prev = p.frames.at((p.r0 + z) % p.R);
  const uint8_t* pprev = p.frames.at((p.r0 + z - 1 + p.R) % p.R);
  const uint32_t* points = p.points + (size_t)z * P;
  const float2* disp = p.disp + (size_t)z * P;
  const uint8_t* status = p.status + (size_t)z * P;
  uint32_t* claims = p.claims + (size_t)z * N * P;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / N;
    const int k = (int)(e - j * N) + 1;
    size_t slot;
    int value;
    uint32_t key;
    if (!splat_item(p, prev, pprev, points, disp, status, j, k, slot, value, key)) continue;
    if (claims[slot] == key) {
      if (p.diff_mode) p.dvals[(size_t)z * N * P + slot] = (int16_t)value;
      else p.svals[(size_t)z * N * P + slot] = (uint8_t)value;
      claims[slot] = 0u;
    }
  }
}

// difference_interp's flow images: min(255, |f_j - f_(j-1)|) (simulate.cpp:226-229)
__global__ void mags_kernel(Ring<const uint8_t> frames, Ring<uint8_t> mags, int R, int slot0, size_t P) {
  const int slot = (slot0 + (int)blockIdx.y) % R;
  const uint8_t* a = frames.at((slot - 1 + R) % R);
  const uint8_t* b = frames.at(slot);
  uint8_t* m = mags.at(slot);
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (size_t)gridDim.x * blockDim.x)
    m[i] = (uint8_t)min(255, abs((int)b[i] - (int)a[i]));
}

__global__ void init_ref_kernel(const uint8_t* __restrict__ f, const float* __restrict__ lut, float* __restrict__ ref,
                                int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) ref[i] = lut[f[i]];
}

// ------------------------------------------------------------ launches

// cudaFuncAttributeMaxDynamicSharedMemorySize is per (function, device): set
// it once per pair, thread-safely (handles on several devices may launch from
// several host threads), and fail loudly if the driver refuses.
void set_max_dynamic_smem(const void* func, int bytes) {
  static std::mutex m;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) throw std::runtime_error("cudaGetDevice failed");
  std::lock_guard<std::mutex> g(m);
  if (done.count({func, dev})) return;
  const cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) throw std::runtime_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
  done.insert({func, dev});
}

template <class Prov, bool kLog, bool kMag, int kW, int kB, int kMinBlocks>
static void launch_chain_k(const ChainParams& p, cudaStream_t s) {
  const size_t sm = (size_t)std::max(p.d.n_links * p.n_pairs, 1) * sizeof(uint32_t);
  auto* k = chain_kernel<Prov, kLog, kMag, kW, kB, kMinBlocks>;
  set_max_dynamic_smem((const void*)k, 96 * 1024);
  k<<<p.n_blocks, 256, sm, s>>>(p);
}

template <class Prov, bool kLog, bool kMag>
static void launch_chain_t(const ChainParams& p, cudaStream_t s) {
  // 2 words x 4 links in flight per warp; 3 blocks of 256 per SM (80 regs).
  // Measured on c2/c5: 1 word x 8 links is within 5% on c2, 8% slower on c5.
  launch_chain_k<Prov, kLog, kMag, 2, 4, 3>(p, s);
}

template <class Prov>
static void launch_chain_mode(const ChainParams& p, cudaStream_t s) {
  if (p.log_mode) {
    if (p.magnitude) launch_chain_t<Prov, true, true>(p, s);
    else launch_chain_t<Prov, true, false>(p, s);
  } else {
    if (p.magnitude) launch_chain_t<Prov, false, true>(p, s);
    else launch_chain_t<Prov, false, false>(p, s);
  }
}

template <bool kLog, bool kMag, int kB, int kW, int kMinB>
static void launch_chain_dense_b(const ChainParams& p, size_t sm, cudaStream_t s) {
  auto* k = p.quadh.base   ? chain_dense_kernel<kLog, kMag, kB, kW, kMinB, 2>
            : p.quadf.base ? chain_dense_kernel<kLog, kMag, kB, kW, kMinB, 1>
                           : chain_dense_kernel<kLog, kMag, kB, kW, kMinB, 0>;
  set_max_dynamic_smem((const void*)k, 96 * 1024);
  k<<<p.n_blocks, 256, sm, s>>>(p);
}

// the tile-staged form (log / linear single mode, tile geometry): shared
// memory = the staging rows only (counts go out per tile row)
template <bool kLog, int kB>
static void launch_chain_dense_tile_b(const ChainParams& p, cudaStream_t s) {
  const size_t sm = (size_t)p.tile_cap_rows * kTilePB;
  const int tiles = (p.wpr / kTileW) * (int)((p.n_words / p.wpr + kTileH - 1) / kTileH);
  if (p.tile_min_blocks >= 4) {
    auto* k = chain_dense_tile_kernel<kLog, kB, 4>;
    set_max_dynamic_smem((const void*)k, (int)sm);
    k<<<tiles, 256, sm, s>>>(p);
  } else {
    auto* k = chain_dense_tile_kernel<kLog, kB, 3>;
    set_max_dynamic_smem((const void*)k, (int)sm);
    k<<<tiles, 256, sm, s>>>(p);
  }
}
template <bool kLog>
static void launch_chain_dense_tile(const ChainParams& p, cudaStream_t s) {
  const int n_int = std::min(p.d.n_links, p.n_interp - p.d.start);
  auto tiles = [&](int b) { return n_int > 0 && n_int % b == 0; };
  if (tiles(8)) launch_chain_dense_tile_b<kLog, 8>(p, s);
  else if (tiles(10)) launch_chain_dense_tile_b<kLog, 10>(p, s);
  else if (tiles(5) && !tiles(4)) launch_chain_dense_tile_b<kLog, 5>(p, s);
  else launch_chain_dense_tile_b<kLog, 4>(p, s);
}

template <bool kLog, bool kMag>
static void launch_chain_dense(const ChainParams& p, size_t sm, cudaStream_t s) {
  // the longest batch that tiles the interior links (more gathers in flight
  // per warp; measured on c2 N=10: batches of 10 vs 5, chain 12.7 -> 12.1
  // us/frame), else batches of 4 with a remainder.  One-word warp tasks
  // (EventEngine::geometry), 3 blocks/SM at 80 regs (4 at 64 regs: c2 chain
  // 12.6 -> 13.1; two-word tasks at 128 regs: c5 782 vs 707 µs/frame)
  const int n_int = std::min(p.d.n_links, p.n_interp - p.d.start);
  auto tiles = [&](int b) { return n_int > 0 && n_int % b == 0; };
  // log single mode, batches of 8: 4 blocks/SM at 64 registers (the level
  // thresholds need fewer registers than the fp32 rule; c5 log chain 604 ->
  // 581 us/frame; the same cap on batches of 4 / 5 / 10 or on linear mode
  // measured equal or slower: c2 log 10.5 -> 11.8 us/frame at batches of 10)
  if (kLog && !kMag && tiles(8)) {
    launch_chain_dense_b<kLog, kMag, 8, 1, 4>(p, sm, s);
    return;
  }
  if (tiles(10)) launch_chain_dense_b<kLog, kMag, 10, 1, 3>(p, sm, s);
  else if (tiles(8)) launch_chain_dense_b<kLog, kMag, 8, 1, 3>(p, sm, s);
  else if (tiles(5) && !tiles(4)) launch_chain_dense_b<kLog, kMag, 5, 1, 3>(p, sm, s);
  else launch_chain_dense_b<kLog, kMag, 4, 1, 3>(p, sm, s);
}

template <bool kLog, bool kMag>
static void launch_chain_sparse(const ChainParams& p, size_t sm, cudaStream_t s) {
  (void)sm;
  auto* k = chain_sparse_kernel<kLog, kMag>;
  cudaMemsetAsync(p.counts, 0, (size_t)std::max(p.d.n_links * p.n_pairs, 1) * p.n_blocks * sizeof(uint32_t), s);
  cudaMemsetAsync(p.sched, 0, sizeof(unsigned int), s);
  // persistent: 3 resident blocks of 8 warps per SM take tasks until done
  const int64_t tasks = (p.n_words + 1) / 2;
  const int64_t blocks = std::min<int64_t>((tasks + kWarpsPerBlock - 1) / kWarpsPerBlock, 148 * 3);
  k<<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, s>>>(p);
}

template <bool kMag>
static void launch_chain_diffinterp(const ChainParams& p, size_t sm, cudaStream_t s) {
  auto* k = chain_diffinterp_kernel<kMag>;
  set_max_dynamic_smem((const void*)k, 96 * 1024);
  k<<<p.n_blocks, 256, sm, s>>>(p);
}

void launch_chain(const ChainParams& p, int provider, cudaStream_t s) {
  if (provider == kProvDiffInterp) {
    const size_t sm = (size_t)std::max(p.d.n_links * p.n_pairs, 1) * sizeof(uint32_t);
    if (p.magnitude) launch_chain_diffinterp<true>(p, sm, s);
    else launch_chain_diffinterp<false>(p, sm, s);
    return;
  }
  if (provider == kProvSparse) {
    const size_t sm = (size_t)std::max(p.d.n_links * p.n_pairs, 1) * sizeof(uint32_t);
    if (p.log_mode) {
      if (p.magnitude) launch_chain_sparse<true, true>(p, sm, s);
      else launch_chain_sparse<true, false>(p, sm, s);
    } else {
      if (p.magnitude) launch_chain_sparse<false, true>(p, sm, s);
      else launch_chain_sparse<false, false>(p, sm, s);
    }
    return;
  }
  if (provider == kProvDenseGrid && p.kc && p.n_interp + 2 <= kMaxParamK && p.quadt.base && !p.magnitude &&
      p.words_per_block == kTileW && p.wpr % kTileW == 0) {
    if (p.log_mode) launch_chain_dense_tile<true>(p, s);
    else launch_chain_dense_tile<false>(p, s);
    return;
  }
  if (provider == kProvDenseGrid && p.kc && p.n_interp + 2 <= kMaxParamK) {
    const size_t sm = (size_t)(p.n_interp + 2) * sizeof(float4) +
                      (size_t)std::max(p.d.n_links * p.n_pairs, 1) * sizeof(uint32_t);
    if (sm <= 96 * 1024) {
      if (p.log_mode) {
        if (p.magnitude) launch_chain_dense<true, true>(p, sm, s);
        else launch_chain_dense<true, false>(p, sm, s);
      } else {
        if (p.magnitude) launch_chain_dense<false, true>(p, sm, s);
        else launch_chain_dense<false, false>(p, sm, s);
      }
      return;
    }
  }
  if (provider == kProvNone && !p.magnitude && p.d.n_links == 1 && p.n_interp == 0 && !p.skip_empty &&
      (size_t)p.n_pairs * sizeof(uint32_t) <= 48 * 1024) {
    // difference_only: the streaming chain
    const size_t sm = (size_t)p.n_pairs * sizeof(uint32_t);
    static const bool no_tma = [] {
      const char* e = std::getenv("EVSIM_DIFF_NO_TMA");
      return e && e[0] == '1';
    }();
    if (!no_tma && chain_diff_tma_ok(p)) {
      const int sb = diff_stage_bytes(p);
      const size_t smt = (size_t)kDiffNB * sb + sm;
      auto* k = p.log_mode ? chain_diff_tma_kernel<true> : chain_diff_tma_kernel<false>;
      set_max_dynamic_smem((const void*)k, 160 * 1024);
      k<<<p.n_blocks, 256, smt, s>>>(p, sb);
      return;
    }
    if (p.log_mode) chain_diff_kernel<true, 16><<<p.n_blocks, 256, sm, s>>>(p);
    else chain_diff_kernel<false, 16><<<p.n_blocks, 256, sm, s>>>(p);
    return;
  }
  switch (provider) {
    case kProvDenseGrid: launch_chain_mode<DenseProvider<false>>(p, s); break;
    case kProvDenseField: launch_chain_mode<DenseProvider<true>>(p, s); break;
    default: launch_chain_mode<NoneProvider>(p, s); break;
  }
}

void launch_segments(const SegParams& p, cudaStream_t s) { segments_kernel<<<1, 1024, 0, s>>>(p); }

void launch_offsets(const OffsetParams& p, cudaStream_t s) {
  if (p.n_rows <= 0) return;
  if (p.n_rows < 4 * 148) offsets_row_kernel<<<p.n_rows, 256, 0, s>>>(p);
  else offsets_kernel<<<(p.n_rows + kWarpsPerBlock - 1) / kWarpsPerBlock, 256, 0, s>>>(p);
}

void launch_segbase(const EmitParams& p, int64_t* segbase, cudaStream_t s) {
  segbase_kernel<<<1, 1024, 0, s>>>(p, segbase);
}

// segbase_kernel then emit_kernel; segbase: [links] int64 scratch
void launch_emit(const EmitParams& p, int64_t* segbase, cudaStream_t s) {
  segbase_kernel<<<1, 1024, 0, s>>>(p, segbase);
  const size_t sm = (size_t)std::max(p.n_links, 1) * (sizeof(int64_t) + sizeof(int));
  set_max_dynamic_smem((const void*)emit_kernel, 144 * 1024);
  emit_kernel<<<p.n_blocks, 256, sm, s>>>(p, segbase);
}

// segbase_kernel then emit_single_kernel over links [g0, g1) (every link
// its own segment, single mode); false when the geometry does not fit a tile
bool launch_emit_single(const EmitParams& p, int64_t* segbase, int g0, int g1, cudaStream_t s) {
  if (p.magnitude || p.words_per_block > 256 || g1 <= g0) return false;
  segbase_kernel<<<1, 1024, 0, s>>>(p, segbase);
  const int bpt = std::max(1, 256 / p.words_per_block);
  const int tiles = (p.n_blocks + bpt - 1) / bpt;
  // links per block: enough blocks to fill the GPU a few times over, each
  // amortising its setup over up to 8 links
  const int n_links = g1 - g0;
  int lpb = 1;
  while (lpb < 8 && (int64_t)tiles * ((n_links + 2 * lpb - 1) / (2 * lpb)) >= 148 * 16) lpb *= 2;
  const int ys = (n_links + lpb - 1) / lpb;
  emit_single_kernel<<<dim3((unsigned)tiles, (unsigned)ys), 256, 0, s>>>(p, segbase, bpt, g0, g1, lpb);
  return true;
}

void launch_unpack_events(const uint32_t* packed, const int64_t* seg_out, int64_t n, void* out24,
                          cudaStream_t s) {
  if (n <= 0) return;
  unpack_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(packed, seg_out, n, (unsigned long long*)out24);
}

void launch_interp_frames(const ChainParams& p, uint8_t* out, cudaStream_t s) {
  dim3 g((p.w + 127) / 128, p.h);
  interp_frames_kernel<<<g, 128, 0, s>>>(p, out);
}

void launch_select(const SelectParams& p, int n_pairs, cudaStream_t s) {
  if (n_pairs <= 0) return;
  select_mask_kernel<<<dim3(p.n_blocks, n_pairs), 256, 0, s>>>(p);
  OffsetParams op{n_pairs, p.n_blocks, p.counts, p.prefix, p.total};
  launch_offsets(op, s);
  select_emit_kernel<<<dim3(p.n_blocks, n_pairs), 256, 0, s>>>(p);
}

void launch_init_ref(const uint8_t* frame, const float* lut, float* ref, int64_t n, cudaStream_t s) {
  init_ref_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(frame, lut, ref, n);
}

void launch_mags(Ring<const uint8_t> frames, Ring<uint8_t> mags, int R, int slot0, int n, size_t P, cudaStream_t s) {
  if (n <= 0) return;
  const unsigned bx = (unsigned)std::min<size_t>((P + 255) / 256, (148 * 8 + n - 1) / n);
  mags_kernel<<<dim3(std::max(bx, 1u), n), 256, 0, s>>>(frames, mags, R, slot0, P);
}

void launch_splat(const SplatParams& p, int max_items, int n_pairs, cudaStream_t s) {
  if (n_pairs <= 0) return;
  int blocks = (max_items + 255) / 256;
  const int cap = (148 * 16 + n_pairs - 1) / n_pairs;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  splat_kernel<<<dim3(blocks, n_pairs), 256, 0, s>>>(p);
  resolve_kernel<<<dim3(blocks, n_pairs), 256, 0, s>>>(p);
}

}  // namespace evsim_gpu
