// event_kernels.cu — interpolation + difference/threshold chain, ordered
// compaction, sparse selection and splat (sm_100a).
//
// Replaces src/simulate.cpp:91-201 and src/core.cpp:5-46 of the reference
// (/root/reference/proj).  Layout: every link of the chain is
// evaluated per pixel in one pass; a warp covers 32 consecutive pixels of one
// row (a "word") and publishes the link's positive / negative crossings as two
// 32-bit ballots.  Events are then written exactly once, contiguously, in the
// reference's order (t, y, x, p) by a scan over (segment, block) counts and a
// ballot/popc expansion.
#include "evsim_device.cuh"
#include "kernels.h"

namespace evsim_gpu {

namespace {

__device__ __forceinline__ const ChainDesc& pick_desc(const int* d_direct, const ChainDesc& full,
                                                      const ChainDesc& direct) {
  return (d_direct && *d_direct == 0) ? direct : full;
}

// Block-wide exclusive scan of one int64 per thread (256 threads).
__device__ __forceinline__ int64_t block_exclusive_scan(int64_t v, int64_t* s_warp, int64_t& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int64_t w = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(kFull, w, o);
      if (lane >= o) w += y;
    }
    if (lane < (int)(blockDim.x >> 5)) s_warp[lane] = w;  // inclusive warp prefix
  }
  __syncthreads();
  total = s_warp[(blockDim.x >> 5) - 1];
  const int64_t before = warp ? s_warp[warp - 1] : 0;
  __syncthreads();
  return before + x - v;
}

// ------------------------------------------------------------ value providers
// value(k) = intensity of chain frame k at this pixel: k = 0 prev,
// k = N+1 curr, 1..N the interpolated / splatted frame.

struct PixelCtx {
  bool valid;  // false for the padding lanes of a row's last word
  int x, y;
  size_t pix;
  float xf, yf;
};

// Dense: flow-based two-sided interpolation, interpolate_frames
// (simulate.cpp:91-121), with the flow either densified from the level-0
// patch grid (flow.cpp:224-245) or read from a caller-supplied field.
template <bool kField>
struct DenseProvider {
  float u, v;
  __device__ __forceinline__ void init(const ChainParams& p, const PixelCtx& c);
  __device__ __forceinline__ int interp(const ChainParams& p, const PixelCtx& c, int k) const {
    const float fwd = __ldg(p.fwd + k);
    const float bwd = __ldg(p.bwd + k);
    const float fp = sample_quad(p.qprev, p.w, p.h, fsub(c.xf, fmul(fwd, u)), fsub(c.yf, fmul(fwd, v)));
    const float fc = sample_quad(p.qcurr, p.w, p.h, fadd(c.xf, fmul(bwd, u)), fadd(c.yf, fmul(bwd, v)));
    const double blend = dadd(dmul(__ldg(p.oma + k), (double)fp), dmul(__ldg(p.alpha + k), (double)fc));
    return lround_pos(blend);
  }
  __device__ __forceinline__ void finish(const ChainParams&, const PixelCtx&) const {}
};

__device__ __forceinline__ void densify_grid(const GridGeom& g, int x, int y, float& u, float& v) {
  const int j = __ldg(g.iy + y);
  const float fy = __ldg(g.wy + y);
  const int i = __ldg(g.ix + x);
  const float fx = __ldg(g.wx + x);
  const int i0 = min(i, g.ncx - 1), i1 = min(i + 1, g.ncx - 1);
  const int j0 = min(j, g.ncy - 1), j1 = min(j + 1, g.ncy - 1);
  const size_t r0 = (size_t)j0 * g.ncx, r1 = (size_t)j1 * g.ncx;
  const float u_top = lerp_ref(__ldg(g.pu + r0 + i0), __ldg(g.pu + r0 + i1), fx);
  const float u_bot = lerp_ref(__ldg(g.pu + r1 + i0), __ldg(g.pu + r1 + i1), fx);
  const float v_top = lerp_ref(__ldg(g.pv + r0 + i0), __ldg(g.pv + r0 + i1), fx);
  const float v_bot = lerp_ref(__ldg(g.pv + r1 + i0), __ldg(g.pv + r1 + i1), fx);
  u = lerp_ref(u_top, u_bot, fy);
  v = lerp_ref(v_top, v_bot, fy);
}

template <>
__device__ __forceinline__ void DenseProvider<false>::init(const ChainParams& p, const PixelCtx& c) {
  densify_grid(p.g0, c.x, c.y, u, v);
}
template <>
__device__ __forceinline__ void DenseProvider<true>::init(const ChainParams& p, const PixelCtx& c) {
  u = __ldg(p.du + c.pix);
  v = __ldg(p.dv + c.pix);
}

// Sparse: intermediate frame k is prev with the winning splat, if any
// (simulate.cpp:167-199).  Consumed claim slots are cleared so the planes are
// all-zero again for the next push.
struct SparseProvider {
  uint32_t tw0, tw1;  // touched bits of frames 1..64 (n_interp <= 64 fast path)
  __device__ __forceinline__ void init(const ChainParams& p, const PixelCtx& c) {
    const size_t P = (size_t)p.w * p.h;
    tw0 = p.n_interp > 0 ? p.touched[c.pix] : 0u;
    tw1 = p.n_interp > 32 ? p.touched[P + c.pix] : 0u;
  }
  __device__ __forceinline__ bool touched_bit(const ChainParams& p, const PixelCtx& c, int k) const {
    const int b = k - 1;
    if (b < 32) return (tw0 >> b) & 1u;
    if (b < 64) return (tw1 >> (b - 32)) & 1u;
    const size_t P = (size_t)p.w * p.h;
    return (p.touched[(size_t)(b >> 5) * P + c.pix] >> (b & 31)) & 1u;
  }
  __device__ __forceinline__ int interp(const ChainParams& p, const PixelCtx& c, int k) const {
    if (!touched_bit(p, c, k)) return p.prev[c.pix];
    const size_t P = (size_t)p.w * p.h;
    const size_t slot = (size_t)(k - 1) * P + c.pix;
    const uint64_t key = p.claims[slot];
    if (c.valid) p.claims_rw[slot] = 0ull;
    const uint32_t j = 0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFull);
    return p.prev[__ldg(p.points + j)];
  }
  __device__ __forceinline__ void finish(const ChainParams& p, const PixelCtx& c) const {
    const size_t P = (size_t)p.w * p.h;
    const int nw = (p.n_interp + 31) >> 5;
    for (int i = 0; i < nw; ++i) {
      const uint32_t t = i == 0 ? tw0 : (i == 1 ? tw1 : p.touched[(size_t)i * P + c.pix]);
      if (t) p.touched_rw[(size_t)i * P + c.pix] = 0u;
    }
  }
};

// No intermediate frames: chains over prev/curr only (difference_only, N = 0).
struct NoneProvider {
  __device__ __forceinline__ void init(const ChainParams&, const PixelCtx&) {}
  __device__ __forceinline__ int interp(const ChainParams& p, const PixelCtx& c, int) const { return p.prev[c.pix]; }
  __device__ __forceinline__ void finish(const ChainParams&, const PixelCtx&) const {}
};

template <class Prov>
__device__ __forceinline__ int frame_value(const ChainParams& p, const Prov& prov, const PixelCtx& c, int k) {
  if (k == 0) return p.prev[c.pix];
  if (k == p.n_interp + 1) return p.curr[c.pix];
  return prov.interp(p, c, k);
}

}  // namespace

// ------------------------------------------------------------ chain kernel
//
// One warp = one 32-pixel word of one row.  For every link of the chain the
// warp evaluates the reference rule per lane (difference_frame +
// threshold_events_into, core.cpp:5-46, or the log rule of DESIGN.md §3),
// ballots the crossings and lane 0 stores the (pos, neg) masks.
template <class Prov, bool kLog, bool kMag>
__global__ void __launch_bounds__(256) chain_kernel(ChainParams p) {
  extern __shared__ uint32_t s_cnt[];  // per-link event counts of this block
  __shared__ float s_lut[256];
  const ChainDesc& d = pick_desc(p.d_direct, p.full, p.direct);
  const int L = d.n_links;
  for (int i = threadIdx.x; i < L; i += blockDim.x) s_cnt[i] = 0;
  if (kLog) s_lut[threadIdx.x] = p.lut[threadIdx.x];
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t wbeg = (int64_t)blockIdx.x * p.words_per_block;
  const int64_t wend = min(wbeg + p.words_per_block, p.n_words);
  for (int64_t wi = wbeg + warp; wi < wend; wi += kWarpsPerBlock) {
    const int row = (int)(wi / p.wpr);
    const int x = (int)(wi - (int64_t)row * p.wpr) * 32 + lane;
    const bool valid = x < p.w;
    PixelCtx c;
    c.valid = valid;
    c.x = valid ? x : p.w - 1;
    c.y = row;
    c.pix = (size_t)row * p.w + c.x;
    c.xf = (float)c.x;
    c.yf = (float)c.y;
    Prov prov;
    prov.init(p, c);

    int before = 0;
    float ref = 0.0f;
    if (kLog) ref = p.ref[c.pix];
    else before = frame_value(p, prov, c, d.start);
    for (int l = 0; l < L; ++l) {
      const int val = frame_value(p, prov, c, d.start + (l + 1) * d.step);
      bool pos, neg;
      int mult = 1;
      if (kLog) {
        const float lk = s_lut[val];
        const float dd = fsub(lk, ref);
        pos = dd > p.c_pos_log;
        neg = !pos && dd < p.c_neg_log;
        if (kMag && (pos || neg)) mult = (int)floorf(__fdiv_rn(dd, pos ? p.c_pos_log : p.c_neg_log));
        if (pos || neg) ref = lk;
      } else {
        const int v = val - before;  // difference_frame, core.cpp:14-15
        pos = v > p.c_pos;           // threshold_events_into, core.cpp:31-43
        neg = !pos && v < p.c_neg;
        if (kMag && (pos || neg)) mult = pos ? v / p.c_pos : v / p.c_neg;
        before = val;
      }
      pos = pos && valid;
      neg = neg && valid;
      const unsigned bp = __ballot_sync(kFull, pos);
      const unsigned bn = __ballot_sync(kFull, neg);
      if (lane == 0) p.masks[(size_t)l * p.n_words + wi] = make_uint2(bp, bn);
      if (kMag) {
        const int m = (pos || neg) ? mult : 0;
        p.mcount[(size_t)l * p.n_words * 32 + wi * 32 + lane] = (uint16_t)m;
        int s = m;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
        if (lane == 0) {
          p.wcount[(size_t)l * p.n_words + wi] = (uint32_t)s;
          if (s) atomicAdd(&s_cnt[l], (uint32_t)s);
        }
      } else if (lane == 0 && (bp | bn)) {
        atomicAdd(&s_cnt[l], (uint32_t)(__popc(bp) + __popc(bn)));
      }
    }
    if (kLog && valid) p.ref[c.pix] = ref;
    if (valid) prov.finish(p, c);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < L; i += blockDim.x) p.counts[(size_t)i * p.n_blocks + blockIdx.x] = s_cnt[i];
}

// ------------------------------------------------------------ scan kernel
//
// Exclusive scan of (segment, block) event counts in segment-major order:
// the offset of block b's events of segment s.  One block of
// 1024 threads; each thread sums a contiguous run of entries.
__device__ __forceinline__ int64_t sub_interval_end(int64_t t0, int64_t t1, int k, int n_steps) {
  // include/evsim/simulate.hpp:15-19
  const int64_t dt = t1 - t0;
  const int64_t num = (int64_t)k * dt;
  return t0 + (num + n_steps - 1) / n_steps;
}

__global__ void __launch_bounds__(1024) scan_kernel(ScanParams p) {
  __shared__ int64_t s_warp[32];
  __shared__ int s_S;
  const ChainDesc& d = pick_desc(p.d_direct, p.full, p.direct);
  if (threadIdx.x == 0) {
    // chain frame timestamps (simulate.cpp:44-69 + sub_interval_end) grouped
    // into runs of equal value
    int S = 0;
    int64_t last = 0;
    for (int l = 0; l < d.n_links; ++l) {
      const int k = d.start + (l + 1) * d.step;
      const int64_t t = k == p.n_interp + 1 ? p.t_curr : sub_interval_end(p.t_prev, p.t_curr, k, p.n_interp + 1);
      if (S > 0 && t == last) {
        p.seg.seg_nlinks[S - 1]++;
      } else {
        p.seg.seg_first[S] = l;
        p.seg.seg_nlinks[S] = 1;
        p.seg.seg_t[S] = t;
        ++S;
      }
      last = t;
    }
    *p.seg.n_segs = S;
    s_S = S;
  }
  __syncthreads();
  const int S = s_S;
  const int64_t T = (int64_t)S * p.n_blocks;
  const int64_t per = (T + blockDim.x - 1) / blockDim.x;
  const int64_t e0 = min((int64_t)threadIdx.x * per, T), e1 = min(e0 + per, T);
  auto val = [&](int64_t e) -> int64_t {
    const int s = (int)(e / p.n_blocks);
    const int b = (int)(e - (int64_t)s * p.n_blocks);
    int64_t v = 0;
    const int k0 = p.seg.seg_first[s], nk = p.seg.seg_nlinks[s];
    for (int k = k0; k < k0 + nk; ++k) v += p.counts[(size_t)k * p.n_blocks + b];
    return v;
  };
  int64_t sum = 0;
  for (int64_t e = e0; e < e1; ++e) sum += val(e);
  // block exclusive scan (1024 threads)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t x = sum;
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int64_t w = s_warp[lane];
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(kFull, w, o);
      if (lane >= o) w += y;
    }
    s_warp[lane] = w;
  }
  __syncthreads();
  int64_t run = (warp ? s_warp[warp - 1] : 0) + x - sum;
  const int64_t total = s_warp[31];
  for (int64_t e = e0; e < e1; ++e) {
    p.offsets[e] = run;
    run += val(e);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    p.seg_out[0] = S;
    *p.total = total;
    if (p.host_total) *(volatile int64_t*)p.host_total = total;
  }
  for (int s = threadIdx.x; s < S; s += blockDim.x) {
    p.seg_out[1 + s] = p.seg.seg_t[s];
    p.seg_out[1 + S + s] = p.offsets[(int64_t)s * p.n_blocks];
  }
  if (threadIdx.x == 0) p.seg_out[1 + 2 * S] = total;
}

// ------------------------------------------------------------ emit kernel
//
// Writes every event once, in the reference's order.  Per segment the block
// walks its words in chunks of 256 (one per thread), scans the per-word event
// counts and expands each word with lanes = pixels: the event of lane l lands
// at base + word_offset + popc(mask & lanemask_lt) — a warp-ballot compaction.
// Segments with several links (equal timestamps, finalize's stable_sort at
// simulate.cpp:36-40) and magnitude mode take the per-lane count path: per
// pixel all negative events precede the positive ones.
__device__ __forceinline__ uint32_t pack_event(int x, int y, bool neg) {
  return (uint32_t)x | ((uint32_t)y << 16) | (neg ? 0x80000000u : 0u);
}

__global__ void __launch_bounds__(256) emit_kernel(EmitParams p) {
  __shared__ int64_t s_warp[kWarpsPerBlock];
  if (*p.total > p.capacity) return;  // host grows the buffer and re-emits
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t wbeg = (int64_t)blockIdx.x * p.words_per_block;
  const int64_t wend = min(wbeg + p.words_per_block, p.n_words);
  const int S = *p.seg.n_segs;
  for (int s = 0; s < S; ++s) {
    int64_t base = p.offsets[(int64_t)s * p.n_blocks + blockIdx.x];
    const int k0 = p.seg.seg_first[s], nk = p.seg.seg_nlinks[s];
    const bool fast = !p.magnitude && nk == 1;
    for (int64_t cbeg = wbeg; cbeg < wend; cbeg += blockDim.x) {
      const int64_t wi = cbeg + threadIdx.x;
      uint32_t pos = 0, all = 0;
      int64_t cnt = 0;
      if (wi < wend) {
        if (fast) {
          const uint2 m = p.masks[(size_t)k0 * p.n_words + wi];
          pos = m.x;
          all = m.x | m.y;
          cnt = __popc(all);
        } else {
          for (int k = k0; k < k0 + nk; ++k) {
            if (p.magnitude) {
              cnt += p.wcount[(size_t)k * p.n_words + wi];
            } else {
              const uint2 m = p.masks[(size_t)k * p.n_words + wi];
              cnt += __popc(m.x | m.y);
            }
          }
        }
      }
      int64_t chunk_total;
      const int64_t off = block_exclusive_scan(cnt, s_warp, chunk_total);
      if (chunk_total > 0) {
        for (int j = 0; j < 32; ++j) {
          const int64_t wij = cbeg + warp * 32 + j;
          if (wij >= wend) break;
          const int64_t cj = __shfl_sync(kFull, cnt, j);
          const int64_t oj = __shfl_sync(kFull, off, j);
          if (cj == 0) continue;
          const int row = (int)(wij / p.wpr);
          const int x = (int)(wij - (int64_t)row * p.wpr) * 32 + lane;
          if (fast) {
            const uint32_t aj = __shfl_sync(kFull, all, j);
            const uint32_t pj = __shfl_sync(kFull, pos, j);
            if ((aj >> lane) & 1u) {
              const int64_t dst = base + oj + __popc(aj & lanemask_lt());
              p.out[dst] = pack_event(x, row, !((pj >> lane) & 1u));
            }
          } else {
            int nneg = 0, npos = 0;
            for (int k = k0; k < k0 + nk; ++k) {
              const uint2 m = p.masks[(size_t)k * p.n_words + wij];
              const int mult = p.magnitude ? (int)p.mcount[(size_t)k * p.n_words * 32 + wij * 32 + lane] : 1;
              if ((m.x >> lane) & 1u) npos += mult;
              if ((m.y >> lane) & 1u) nneg += mult;
            }
            int incl = nneg + npos;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int y = __shfl_up_sync(kFull, incl, o);
              if (lane >= o) incl += y;
            }
            int64_t dst = base + oj + incl - (nneg + npos);
            for (int q = 0; q < nneg; ++q) p.out[dst++] = pack_event(x, row, true);
            for (int q = 0; q < npos; ++q) p.out[dst++] = pack_event(x, row, false);
          }
        }
      }
      base += chunk_total;
    }
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
  DenseProvider<true> prov;
  prov.init(p, c);
  const size_t P = (size_t)p.w * p.h;
  for (int k = 1; k <= p.n_interp; ++k) out[(size_t)(k - 1) * P + c.pix] = (uint8_t)prov.interp(p, c, k);
}

// ------------------------------------------------------------ sparse selection
// |curr - prev| > sel in scan order (simulate.cpp:149-159); log mode:
// |L(curr) - L(prev)| > sel_log.
__global__ void __launch_bounds__(256) select_mask_kernel(SelectParams p) {
  __shared__ uint32_t s_cnt;
  __shared__ float s_lut[256];
  if (threadIdx.x == 0) s_cnt = 0;
  if (p.log_mode) s_lut[threadIdx.x] = p.lut[threadIdx.x];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t wbeg = (int64_t)blockIdx.x * p.words_per_block;
  const int64_t wend = min(wbeg + p.words_per_block, p.n_words);
  for (int64_t wi = wbeg + warp; wi < wend; wi += kWarpsPerBlock) {
    const int row = (int)(wi / p.wpr);
    const int x = (int)(wi - (int64_t)row * p.wpr) * 32 + lane;
    bool take = false;
    if (x < p.w) {
      const size_t i = (size_t)row * p.w + x;
      const int a = p.prev[i], b = p.curr[i];
      if (p.log_mode) take = fabsf(fsub(s_lut[b], s_lut[a])) > p.sel_log;
      else take = abs(b - a) > p.sel;
    }
    const unsigned m = __ballot_sync(kFull, take);
    if (lane == 0) {
      p.masks[wi] = m;
      if (m) atomicAdd(&s_cnt, (uint32_t)__popc(m));
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) p.counts[blockIdx.x] = s_cnt;
}

// Compact the selection into pixel indices (scan order).  offsets from scan_kernel.
__global__ void __launch_bounds__(256) select_emit_kernel(SelectParams p, const int64_t* __restrict__ total) {
  __shared__ int64_t s_warp[kWarpsPerBlock];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (blockIdx.x == 0 && threadIdx.x == 0) *p.n_points = (int)*total;
  const int64_t wbeg = (int64_t)blockIdx.x * p.words_per_block;
  const int64_t wend = min(wbeg + p.words_per_block, p.n_words);
  int64_t base = p.offsets[blockIdx.x];
  for (int64_t cbeg = wbeg; cbeg < wend; cbeg += blockDim.x) {
    const int64_t wi = cbeg + threadIdx.x;
    const uint32_t m = wi < wend ? p.masks[wi] : 0u;
    int64_t tot;
    const int64_t off = block_exclusive_scan(__popc(m), s_warp, tot);
    if (tot > 0) {
      for (int j = 0; j < 32; ++j) {
        const int64_t wij = cbeg + warp * 32 + j;
        if (wij >= wend) break;
        const uint32_t mj = __shfl_sync(kFull, m, j);
        const int64_t oj = __shfl_sync(kFull, off, j);
        if (!mj) continue;
        if ((mj >> lane) & 1u) {
          const int row = (int)(wij / p.wpr);
          const int x = (int)(wij - (int64_t)row * p.wpr) * 32 + lane;
          p.points[base + oj + __popc(mj & lanemask_lt())] = (uint32_t)row * (uint32_t)p.w + (uint32_t)x;
        }
      }
    }
    base += tot;
  }
}

// ------------------------------------------------------------ sparse splat
// One thread per (point, k): simulate.cpp:175-199.  The claim rule (first
// claim, replaced only by a strictly larger change) selects, per target pixel,
// the point with the largest change and, among equals, the smallest scan
// index j: an atomicMax on (change << 32) | (~j).
__global__ void splat_kernel(SplatParams p) {
  const int64_t M = *p.n_points;
  const int N = p.n_interp;
  const int64_t total = M * N;
  const size_t P = (size_t)p.w * p.h;
  const float denom = (float)(N + 1);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / N;
    const int k = (int)(e - j * N) + 1;
    if (!p.status[j]) continue;
    const uint32_t src = p.points[j];
    const int px = (int)(src % (uint32_t)p.w), py = (int)(src / (uint32_t)p.w);
    const float alpha = __fdiv_rn((float)k, denom);
    const float2 d = p.disp[j];
    const int tx = lroundf_ref(fadd((float)px, fmul(alpha, d.x)));
    const int ty = lroundf_ref(fadd((float)py, fmul(alpha, d.y)));
    if (tx < 0 || tx >= p.w || ty < 0 || ty >= p.h) continue;
    const size_t idx = (size_t)ty * p.w + tx;
    const int value = p.prev[src];
    const int change = abs(value - (int)p.prev[idx]);
    const unsigned long long key = ((unsigned long long)change << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)j);
    atomicMax((unsigned long long*)&p.claims[(size_t)(k - 1) * P + idx], key);
    atomicOr(&p.touched[(size_t)((k - 1) >> 5) * P + idx], 1u << ((k - 1) & 31));
  }
}

// ------------------------------------------------------------ launches

template <class Prov, bool kLog, bool kMag>
static void launch_chain_t(const ChainParams& p, cudaStream_t s) {
  const int links = max(p.full.n_links, p.direct.n_links);
  chain_kernel<Prov, kLog, kMag><<<p.n_blocks, 256, (size_t)max(links, 1) * sizeof(uint32_t), s>>>(p);
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

void launch_chain(const ChainParams& p, int provider, cudaStream_t s) {
  switch (provider) {
    case kProvDenseGrid: launch_chain_mode<DenseProvider<false>>(p, s); break;
    case kProvSparse: launch_chain_mode<SparseProvider>(p, s); break;
    case kProvDenseField: launch_chain_mode<DenseProvider<true>>(p, s); break;
    default: launch_chain_mode<NoneProvider>(p, s); break;
  }
}

void launch_scan(const ScanParams& p, cudaStream_t s) { scan_kernel<<<1, 1024, 0, s>>>(p); }

void launch_emit(const EmitParams& p, cudaStream_t s) { emit_kernel<<<p.n_blocks, 256, 0, s>>>(p); }

void launch_unpack_events(const uint32_t* packed, const int64_t* seg_out, int64_t n, void* out24,
                          cudaStream_t s) {
  if (n <= 0) return;
  unpack_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(packed, seg_out, n, (unsigned long long*)out24);
}

void launch_interp_frames(const ChainParams& p, uint8_t* out, cudaStream_t s) {
  dim3 g((p.w + 127) / 128, p.h);
  interp_frames_kernel<<<g, 128, 0, s>>>(p, out);
}

void launch_select(const SelectParams& p, cudaStream_t s) { select_mask_kernel<<<p.n_blocks, 256, 0, s>>>(p); }

__global__ void init_ref_kernel(const uint8_t* __restrict__ f, const float* __restrict__ lut, float* __restrict__ ref,
                                int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) ref[i] = lut[f[i]];
}

void launch_init_ref(const uint8_t* frame, const float* lut, float* ref, int64_t n, cudaStream_t s) {
  init_ref_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(frame, lut, ref, n);
}

void launch_select_emit(const SelectParams& p, const int64_t* total, cudaStream_t s) {
  select_emit_kernel<<<p.n_blocks, 256, 0, s>>>(p, total);
}

void launch_splat(const SplatParams& p, int max_items, cudaStream_t s) {
  int blocks = (max_items + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  splat_kernel<<<blocks, 256, 0, s>>>(p);
}

}  // namespace evsim_gpu
