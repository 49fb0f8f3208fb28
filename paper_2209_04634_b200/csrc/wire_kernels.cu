// wire_kernels.cu — the compact lossless event wire format (sm_100a).
//
// The reference hands its caller a std::vector<Event> of 24-byte records
// (include/evsim/types.hpp:54-80); on dense streams (c5: 67-160 M events per
// frame) that is 1.6-3.8 GB per frame, far beyond PCIe.  The wire format
// carries the same events losslessly in the chain's own structure:
//
//   plane[g][w]   u32 per (link, 32-pixel word): bit i = an event at pixel
//                 x = 32 * (w % wpr) + i, y = row0 + w / wpr
//   polarity      one bit per event, in (link, word, bit) order, 1 = the
//                 event is negative, packed LSB-first into u32 words from
//                 link_bit[g] on
//
// i.e. 1 bit per pixel-link plus 1 bit per event (c5 log: 34 + 8 MB per frame
// against 269 MB of packed 4-byte events).  The events of a link in the
// reference's order (y, x) are the set bits of its plane in word order
// (threshold_events_into's scan order, src/core.cpp:21-46); equal-timestamp
// links form one reference segment whose events finalize() orders (y, x, p)
// (src/simulate.cpp:36-40) — the host unpacker merges those.
//
// wire_linkbase_kernel: first polarity bit of every link of the launch
//   (exclusive scan of the chain's per-link totals, starting at the call's
//   running bit counter rounded up to a u32 boundary, so a launch never
//   shares a polarity word with the previous one — its words can be
//   downloaded while the next launch runs).
// wire_kernel: one CTA per (tile of chain blocks, link): planes = pos | neg,
//   polarity bits = compress(neg, plane) per word, placed by a block scan of
//   the words' popcounts at the tile's bit offset (the chain's per-(link,
//   block) exclusive prefix) and staged in shared memory; interior u32 words
//   are stored, the two boundary words OR-ed (the buffer is zeroed per call).
#include "evsim_device.cuh"
#include "kernels.h"

namespace evsim_gpu {

namespace {

// bits of x at the set positions of m, packed to the low end (PEXT);
// Hacker's Delight 7-4, five parallel-suffix rounds.
__device__ __forceinline__ uint32_t compress32(uint32_t x, uint32_t m) {
  x &= m;
  uint32_t mk = ~m << 1;
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    uint32_t mp = mk ^ (mk << 1);
    mp ^= mp << 2;
    mp ^= mp << 4;
    mp ^= mp << 8;
    mp ^= mp << 16;
    const uint32_t mv = mp & m;
    m = (m ^ mv) | (mv >> (1 << i));
    const uint32_t t = x & mv;
    x = (x ^ t) | (t >> (1 << i));
    mk &= ~mp;
  }
  return x;
}

template <class T>
__device__ __forceinline__ T block_scan_excl(T v, T* s_warp, T& total) {
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

}  // namespace

__global__ void __launch_bounds__(1024) wire_linkbase_kernel(WireParams p) {
  __shared__ int64_t s_warp[32];
  const int64_t start = (*p.bit_base + 31) & ~(int64_t)31;
  int64_t carry = start;
  for (int g0 = 0; g0 < p.n_links; g0 += blockDim.x) {
    const int g = g0 + threadIdx.x;
    const int64_t t = g < p.n_links ? p.link_total[g] : 0;
    int64_t chunk;
    const int64_t excl = block_scan_excl(t, s_warp, chunk);
    if (g < p.n_links) {
      p.link_bit[g] = carry + excl;
      p.link_count[g] = t;
    }
    carry += chunk;
  }
  if (threadIdx.x == 0) *p.bit_base = carry;
}

__global__ void __launch_bounds__(256) wire_kernel(WireParams p) {
  __shared__ uint32_t s_bits[256 + 2];
  __shared__ int s_warp[8];
  const int g = blockIdx.y;
  const int b0 = blockIdx.x * p.blocks_per_tile;
  const int64_t w0 = (int64_t)b0 * p.words_per_block;
  const int64_t w1 = min((int64_t)(b0 + p.blocks_per_tile) * p.words_per_block, p.n_words);
  const uint2* masks = p.masks + (size_t)g * p.n_words;
  uint32_t* planes = p.planes + (size_t)g * p.n_words;
  // global polarity bit of the tile's first event
  int64_t bit = p.link_bit[g] + p.prefix[(size_t)g * p.n_blocks + b0];
  for (int64_t c0 = w0; c0 < w1; c0 += 256) {
    const int64_t w = c0 + threadIdx.x;
    uint32_t all = 0, neg = 0;
    if (w < w1) {
      const uint2 m = masks[w];
      all = m.x | m.y;
      neg = m.y;
      planes[w] = all;
    }
    const int cnt = __popc(all);
    int total;
    const int excl = block_scan_excl(cnt, s_warp, total);
    if (total == 0) continue;  // uniform
    const int s0 = (int)(bit & 31);
    const int nq = (s0 + total + 31) >> 5;
    for (int q = threadIdx.x; q < nq; q += 256) s_bits[q] = 0u;
    __syncthreads();
    if (cnt) {
      const uint32_t bits = compress32(neg, all);
      const int pos = s0 + excl;
      const int q = pos >> 5, r = pos & 31;
      atomicOr(&s_bits[q], bits << r);
      if (r + cnt > 32) atomicOr(&s_bits[q + 1], bits >> (32 - r));
    }
    __syncthreads();
    uint32_t* dst = p.pol + (bit >> 5);
    for (int q = threadIdx.x; q < nq; q += 256) {
      const uint32_t v = s_bits[q];
      if (q == 0 || q == nq - 1) {
        if (v) atomicOr(dst + q, v);
      } else {
        dst[q] = v;
      }
    }
    bit += total;
    __syncthreads();
  }
}

void launch_wire(const WireParams& p, cudaStream_t s) {
  if (p.n_links <= 0) return;
  wire_linkbase_kernel<<<1, 1024, 0, s>>>(p);
  const int tiles = (p.n_blocks + p.blocks_per_tile - 1) / p.blocks_per_tile;
  wire_kernel<<<dim3((unsigned)tiles, (unsigned)p.n_links), 256, 0, s>>>(p);
}

}  // namespace evsim_gpu
