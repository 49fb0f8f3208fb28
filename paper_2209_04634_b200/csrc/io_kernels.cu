// io_kernels.cu — the data formats either side of the path:
// frame ingestion (BT.601 luma + bilinear resize, src/io.cpp:41-70), the
// .evs event records (src/io.cpp:148-170) and the event metrics
// (src/metrics.cpp:7-69), on the device.
#include <algorithm>

#include "evsim_device.cuh"
#include "kernels.h"

namespace evsim_gpu {

namespace {

// luma_bt601 (io.cpp:41-43): integer, exact
__global__ void luma_kernel(const uint8_t* __restrict__ rgb, uint8_t* __restrict__ out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = rgb[3 * i], g = rgb[3 * i + 1], b = rgb[3 * i + 2];
    out[i] = (uint8_t)((299 * r + 587 * g + 114 * b + 500) / 1000);
  }
}

// resize_bilinear (io.cpp:45-70): the reference's fp32 steps, lroundf
__global__ void resize_kernel(const uint8_t* __restrict__ src, int w, int h, uint8_t* __restrict__ dst, int tw,
                              int th) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  const int f = blockIdx.z;
  if (x >= tw) return;
  const uint8_t* s = src + (size_t)f * w * h;
  const float sx_ratio = __fdiv_rn((float)w, (float)tw);
  const float sy_ratio = __fdiv_rn((float)h, (float)th);
  const float sy = clamp_ref(fsub(fmul(fadd((float)y, 0.5f), sy_ratio), 0.5f), 0.0f, (float)(h - 1));
  const int y0 = (int)sy;
  const int y1 = min(y0 + 1, h - 1);
  const float fy = fsub(sy, (float)y0);
  const float sx = clamp_ref(fsub(fmul(fadd((float)x, 0.5f), sx_ratio), 0.5f), 0.0f, (float)(w - 1));
  const int x0 = (int)sx;
  const int x1 = min(x0 + 1, w - 1);
  const float fx = fsub(sx, (float)x0);
  const uint8_t* r0 = s + (size_t)y0 * w;
  const uint8_t* r1 = s + (size_t)y1 * w;
  const float top = lerp_ref((float)r0[x0], (float)r0[x1], fx);
  const float bot = lerp_ref((float)r1[x0], (float)r1[x1], fx);
  dst[(size_t)f * tw * th + (size_t)y * tw + x] = (uint8_t)lroundf_ref(lerp_ref(top, bot, fy));
}

// .evs records (io.cpp:158-165): x u16, y u16, t u64, p i8, little endian, 13 B
__global__ void evs_kernel(const uint32_t* __restrict__ packed, const int64_t* __restrict__ seg_out, int64_t n,
                           uint8_t* __restrict__ out) {
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
  const uint64_t t = (uint64_t)st[lo];
  uint8_t* o = out + 13 * i;
  o[0] = (uint8_t)(e & 0xFF);
  o[1] = (uint8_t)((e >> 8) & 0xFF);
  o[2] = (uint8_t)((e >> 16) & 0xFF);
  o[3] = (uint8_t)((e >> 24) & 0x7F);
#pragma unroll
  for (int b = 0; b < 8; ++b) o[4 + b] = (uint8_t)(t >> (8 * b));
  o[12] = (e >> 31) ? 0xFF : 0x01;
}

// per-pixel event counts of 24-byte evsim_event records
__global__ void count_kernel(const evsim_event* __restrict__ ev, int64_t n, int w, uint32_t* __restrict__ counts) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&counts[(size_t)ev[i].y * w + ev[i].x], 1u);
}

// accumulate (metrics.cpp:41-69): polarity bits per pixel over [t0, t1);
// none / positive / negative / both is order-independent, so an atomicOr
// of (positive = 1, negative = 2) gives exactly the reference's class.
__global__ void accumulate_kernel(const evsim_event* __restrict__ ev, int64_t n, int w, int64_t t0, int64_t t1,
                                  uint32_t* __restrict__ bits) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const evsim_event e = ev[i];
    if (e.t < t0 || e.t >= t1) continue;
    atomicOr(&bits[(size_t)e.y * w + e.x], e.p > 0 ? 1u : 2u);
  }
}

__global__ void classes_kernel(const uint32_t* __restrict__ bits, uint8_t* __restrict__ out, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (uint8_t)bits[i];  // 0 none, 1 positive, 2 negative, 3 both (PixelClass)
}

unsigned grid_for(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); }

}  // namespace

void launch_luma(const uint8_t* rgb, uint8_t* out, int64_t n, cudaStream_t s) {
  luma_kernel<<<grid_for(n), 256, 0, s>>>(rgb, out, n);
}
void launch_resize(const uint8_t* src, int w, int h, uint8_t* dst, int tw, int th, int n_frames, cudaStream_t s) {
  resize_kernel<<<dim3((tw + 127) / 128, th, n_frames), 128, 0, s>>>(src, w, h, dst, tw, th);
}
void launch_evs_records(const uint32_t* packed, const int64_t* seg_out, int64_t n, uint8_t* out, cudaStream_t s) {
  if (n > 0) evs_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(packed, seg_out, n, out);
}
void launch_event_counts(const evsim_event* ev, int64_t n, int w, uint32_t* counts, cudaStream_t s) {
  if (n > 0) count_kernel<<<grid_for(n), 256, 0, s>>>(ev, n, w, counts);
}
void launch_accumulate(const evsim_event* ev, int64_t n, int w, int64_t t0, int64_t t1, uint32_t* bits,
                       uint8_t* classes, int64_t P, cudaStream_t s) {
  if (n > 0) accumulate_kernel<<<grid_for(n), 256, 0, s>>>(ev, n, w, t0, t1, bits);
  classes_kernel<<<(unsigned)((P + 255) / 256), 256, 0, s>>>(bits, classes, P);
}

}  // namespace evsim_gpu

namespace evsim_gpu {

// ------------------------------------------------------------ merged output
// Segment s of a push (records [off[s], off[s+1]) of its packed stream) to
// dst + dst_off[s]: one block row per segment, 4096 records per block,
// coalesced on both sides.  dst may be peer memory (NVLink P2P / CUDA IPC):
// the ranks of a multi-GPU run place their bands / streams into rank 0's
// merged buffer at the offsets an all-gather of counts gave.
__global__ void place_kernel(const uint32_t* __restrict__ src, const int64_t* __restrict__ off,
                             const int64_t* __restrict__ dst_off, uint32_t* __restrict__ dst) {
  const int s = blockIdx.y;
  const int64_t a = off[s], n = off[s + 1] - a;
  uint32_t* d = dst + dst_off[s];
  for (int64_t i = (int64_t)blockIdx.x * 4096 + threadIdx.x; i < n && i < (int64_t)(blockIdx.x + 1) * 4096;
       i += blockDim.x)
    d[i] = src[a + i];
}

void launch_place(const uint32_t* src, const int64_t* off, const int64_t* dst_off, int n_segs, int64_t max_len,
                  uint32_t* dst, cudaStream_t s) {
  if (n_segs <= 0 || max_len <= 0) return;
  const unsigned gx = (unsigned)((max_len + 4095) / 4096);
  place_kernel<<<dim3(gx, (unsigned)n_segs), 256, 0, s>>>(src, off, dst_off, dst);
}

}  // namespace evsim_gpu

namespace evsim_gpu {

// ------------------------------------------------------------ core.hpp free functions
// difference_frame (core.cpp:5-19): curr - prev per pixel, int16.
__global__ void difference_kernel(const uint8_t* __restrict__ prev, const uint8_t* __restrict__ curr,
                                  int16_t* __restrict__ out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int16_t)((int)curr[i] - (int)prev[i]);
}

// threshold_events_into (core.cpp:21-46) over a caller's difference values:
// a pixel v > c_pos emits count = (magnitude ? v / c_pos : 1) positive
// events, v < c_neg count = (magnitude ? v / c_neg : 1) negative ones, in
// scan order.  Tiles of kThrTile pixels per block; kThrPer consecutive pixels
// per thread.
constexpr int kThrPer = 8, kThrTile = 256 * kThrPer;
__device__ __forceinline__ int thr_count(int v, int c_pos, int c_neg, int mag) {
  if (v > c_pos) return mag ? v / c_pos : 1;
  if (v < c_neg) return mag ? v / c_neg : 1;
  return 0;
}

__global__ void __launch_bounds__(256) threshold_count_kernel(const int16_t* __restrict__ v, int64_t n, int c_pos,
                                                              int c_neg, int mag, int64_t* __restrict__ tile_total) {
  __shared__ int64_t s_warp[8];
  const int64_t i0 = (int64_t)blockIdx.x * kThrTile + (int64_t)threadIdx.x * kThrPer;
  int64_t c = 0;
#pragma unroll
  for (int j = 0; j < kThrPer; ++j)
    if (i0 + j < n) c += thr_count(v[i0 + j], c_pos, c_neg, mag);
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
  if ((threadIdx.x & 31) == 0) s_warp[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int k = 0; k < 8; ++k) t += s_warp[k];
    tile_total[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(256) threshold_emit_kernel(const int16_t* __restrict__ v, int64_t n, int w,
                                                             int c_pos, int c_neg, int mag, int64_t t,
                                                             const int64_t* __restrict__ tile_off,
                                                             evsim_event* __restrict__ out) {
  __shared__ int64_t s_warp[8];
  const int64_t i0 = (int64_t)blockIdx.x * kThrTile + (int64_t)threadIdx.x * kThrPer;
  int cnt[kThrPer];
  int64_t c = 0;
#pragma unroll
  for (int j = 0; j < kThrPer; ++j) {
    cnt[j] = i0 + j < n ? thr_count(v[i0 + j], c_pos, c_neg, mag) : 0;
    c += cnt[j];
  }
  // exclusive block scan of the per-thread counts
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int64_t incl = c;
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_warp[wid] = incl;
  __syncthreads();
  int64_t base = tile_off[blockIdx.x];
  for (int k = 0; k < wid; ++k) base += s_warp[k];
  int64_t o = base + incl - c;
#pragma unroll
  for (int j = 0; j < kThrPer; ++j) {
    if (!cnt[j]) continue;
    const int64_t i = i0 + j;
    const int y = (int)(i / w), x = (int)(i - (int64_t)y * w);
    const int8_t p = v[i] > c_pos ? 1 : -1;
    for (int k = 0; k < cnt[j]; ++k) {
      evsim_event e;
      e.x = (uint16_t)x;
      e.y = (uint16_t)y;
      e.t = t;
      e.p = p;
      out[o++] = e;
    }
  }
}

void launch_difference(const uint8_t* prev, const uint8_t* curr, int16_t* out, int64_t n, cudaStream_t s) {
  if (n > 0) difference_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 32), 256, 0, s>>>(prev, curr, out, n);
}
int64_t threshold_tiles(int64_t n) { return (n + kThrTile - 1) / kThrTile; }
void launch_threshold_count(const int16_t* v, int64_t n, int c_pos, int c_neg, int mag, int64_t* tile_total,
                            cudaStream_t s) {
  if (n > 0) threshold_count_kernel<<<(unsigned)threshold_tiles(n), 256, 0, s>>>(v, n, c_pos, c_neg, mag, tile_total);
}
void launch_threshold_emit(const int16_t* v, int64_t n, int w, int c_pos, int c_neg, int mag, int64_t t,
                           const int64_t* tile_off, evsim_event* out, cudaStream_t s) {
  if (n > 0)
    threshold_emit_kernel<<<(unsigned)threshold_tiles(n), 256, 0, s>>>(v, n, w, c_pos, c_neg, mag, t, tile_off, out);
}

}  // namespace evsim_gpu
