// flow_kernels.cu — image pyramid, dense patch-grid Lucas–Kanade, sparse
// pyramidal Lucas–Kanade (sm_100a).
//
// Replaces src/flow.cpp of the reference (/root/reference/proj).  Every
// float/double operation keeps the reference's operation order and rounding
// (see evsim_device.cuh); fp64 sums that are not exact are accumulated in the
// reference's k-order by one thread per patch / point, so results are
// bit-identical.
#include "evsim_device.cuh"
#include "kernels.h"

namespace evsim_gpu {

// ---------------------------------------------------------------- pyramid

// One pyramid level of one frame: the fp32 level image (to_float /
// downsample, flow.cpp:23-42) and its QUAD image — per pixel the four taps
// sample() reads (flow.cpp:45-57): (x0,y0) (x1,y0) (x0,y1) (x1,y1) with the
// replicate clamp — so a bilinear sample is one 16-byte gather.  Level 0 also
// writes the u8 quad used by sample_u8 in the interpolation.
__device__ __forceinline__ float level_value(const uint8_t* __restrict__ f0, const float* __restrict__ src,
                                             LevelDims sd, int x, int y, bool level0, bool from_u8) {
  if (level0) return (float)f0[(size_t)y * sd.w + x];
  // downsample  flow.cpp:30-42: 0.25f * (((a + b) + c) + d), odd edges replicate
  const int x0 = 2 * x, y0 = 2 * y;
  const int x1 = min(2 * x + 1, sd.w - 1);
  const int y1 = min(2 * y + 1, sd.h - 1);
  if (from_u8) {  // level 1 straight from the u8 frame (level 0 = to_float of it)
    const uint8_t* r0 = f0 + (size_t)y0 * sd.w;
    const uint8_t* r1 = f0 + (size_t)y1 * sd.w;
    return fmul(0.25f, fadd(fadd(fadd((float)r0[x0], (float)r0[x1]), (float)r1[x0]), (float)r1[x1]));
  }
  const float* r0 = src + (size_t)y0 * sd.w;
  const float* r1 = src + (size_t)y1 * sd.w;
  return fmul(0.25f, fadd(fadd(fadd(r0[x0], r0[x1]), r1[x0]), r1[x1]));
}

constexpr int kPyrRows = 8;  // rows per block: fewer, longer-lived blocks (block launch rate bound)

__global__ void pyramid_level_kernel(PyramidParams p, int l) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const LevelDims dd = p.dims[l];
  if (x >= dd.w) return;
  const int slot = (p.slot0 + (int)blockIdx.z) % p.R;
  const bool level0 = l == 0;
  // u8_level0: level 0 lives only as the u8 frame / quad (the dense solver
  // reads those); level 1 downsamples the bytes directly
  const bool from_u8 = l == 1 && p.u8_level0;
  const uint8_t* f0 = p.frames.at(slot);
  const float* src = (level0 || from_u8) ? nullptr : p.pyr[l - 1].at(slot);
  const int x1 = min(x + 1, dd.w - 1);
  // level-0 reads the u8 frame at the level's own coordinates
  const LevelDims rd = level0 ? dd : p.dims[l - 1];
  float* pyr = p.pyr[l].at(slot);
  float4* qpyr = p.qpyr[l].at(slot);
  uint32_t* qu8 = (level0 && p.quad_u8.base) ? p.quad_u8.at(slot) : nullptr;
  const int yb = blockIdx.y * kPyrRows, ye = min(yb + kPyrRows, dd.h);
  // sparse: the template texels (value, gx, gy) of this level come out of
  // the same pass — gradients (flow.cpp:60-73) from the row above / below and
  // the left / right neighbours, all replicate-clamped
  float4* tex = p.tex[l].base ? p.tex[l].at(slot) : nullptr;
  // sparse with a u8 level 0: the level-0 texels packed into one word
  // (value, a10 - left, a01 - up: integers in [-255, 255], so gx = 0.5f *
  // (a10 - left) is recovered exactly)
  uint32_t* t8 = (level0 && p.tex8.base) ? p.tex8.at(slot) : nullptr;
  const int xm = max(x - 1, 0);
  float a00 = level_value(f0, src, rd, x, yb, level0, from_u8);
  float a10 = level_value(f0, src, rd, x1, yb, level0, from_u8);
  float up = (tex || t8) ? level_value(f0, src, rd, x, max(yb - 1, 0), level0, from_u8) : 0.0f;
  for (int y = yb; y < ye; ++y) {
    const int y1 = min(y + 1, dd.h - 1);
    const float a01 = level_value(f0, src, rd, x, y1, level0, from_u8);
    const float a11 = level_value(f0, src, rd, x1, y1, level0, from_u8);
    const size_t i = (size_t)y * dd.w + x;
    if (!(level0 && p.u8_level0)) {
      pyr[i] = a00;
      qpyr[i] = make_float4(a00, a10, a01, a11);
    }
    if (qu8) qu8[i] = (uint32_t)a00 | ((uint32_t)a10 << 8) | ((uint32_t)a01 << 16) | ((uint32_t)a11 << 24);
    if (tex) {
      const float left = level_value(f0, src, rd, xm, y, level0, from_u8);
      tex[i] = make_float4(a00, fmul(0.5f, fsub(a10, left)), fmul(0.5f, fsub(a01, up)), 0.0f);
      up = a00;
    } else if (t8) {
      const float left = level_value(f0, src, rd, xm, y, level0, from_u8);
      const uint32_t dx = (uint32_t)((int)a10 - (int)left) & 0x1FFu, dy = (uint32_t)((int)a01 - (int)up) & 0x1FFu;
      t8[i] = (uint32_t)a00 | (dx << 8) | (dy << 17);
      up = a00;
    }
    a00 = a01;  // the next row's top taps are this row's bottom taps
    a10 = a11;
  }
}

// Level 0 of the dense path when it is only the u8 quad image (u8_level0,
// no texels): four pixels per thread from one aligned word per row (the next
// column's byte from the neighbouring lane), one 16-byte store per row.
// Needs w % 4 == 0; same bytes as pyramid_level_kernel's qu8 output.
// kTex (sparse): also the packed level-0 texels (pyramid_level_kernel's t8
// words): left neighbour from the previous lane's word, the row above
// carried from the previous iteration (both replicate-clamped).
template <bool kTex>
__global__ void quad_level0_kernel(PyramidParams p) {
  const int w = p.dims[0].w, h = p.dims[0].h;
  const int slot = (p.slot0 + (int)blockIdx.z) % p.R;
  const uint8_t* f = p.frames.at(slot);
  uint32_t* q = p.quad_u8.at(slot);
  uint32_t* t8 = kTex ? p.tex8.at(slot) : nullptr;
  const int x4 = 4 * (int)(blockIdx.x * blockDim.x + threadIdx.x);
  const int lane = threadIdx.x & 31;
  const bool in = x4 < w, last = x4 + 4 >= w;  // last: column x4 + 4 replicates x4 + 3
  const int yb = blockIdx.y * kPyrRows, ye = min(yb + kPyrRows, h);
  auto load = [&](int y, uint32_t& wd, uint32_t& nb) {
    const uint32_t* row = reinterpret_cast<const uint32_t*>(f + (size_t)y * w) + (x4 >> 2);
    wd = in ? __ldg(row) : 0u;
    uint32_t nx = __shfl_down_sync(kFull, wd, 1);
    if (lane == 31 && !last) nx = __ldg(row + 1);
    nb = last ? (wd >> 24) : (nx & 0xFFu);
  };
  uint32_t w0, n0, w1, n1, wm = 0u, nm;
  load(yb, w0, n0);
  if (kTex) load(max(yb - 1, 0), wm, nm);
  for (int y = yb; y < ye; ++y) {
    load(min(y + 1, h - 1), w1, n1);
    uint32_t pb = 0u;  // byte x4 - 1 of row y (replicate at x = 0)
    if (kTex) {
      const uint32_t prv = __shfl_up_sync(kFull, w0, 1);
      if (lane == 0 && x4 > 0) pb = (uint32_t)__ldg(f + (size_t)y * w + x4 - 1);
      else pb = x4 == 0 ? (w0 & 0xFFu) : (prv >> 24);
    }
    if (in) {
      const uint32_t t0 = __byte_perm(w0, n0, 0x0043), t1 = __byte_perm(w1, n1, 0x0043);
      const uint4 o = make_uint4(__byte_perm(w0, w1, 0x5410), __byte_perm(w0, w1, 0x6521),
                                 __byte_perm(w0, w1, 0x7632), __byte_perm(t0, t1, 0x5410));
      *reinterpret_cast<uint4*>(q + (size_t)y * w + x4) = o;
      if (kTex) {
        uint32_t tw[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int v = (int)((w0 >> (8 * j)) & 0xFFu);
          const int right = j < 3 ? (int)((w0 >> (8 * j + 8)) & 0xFFu) : (int)n0;
          const int left = j > 0 ? (int)((w0 >> (8 * j - 8)) & 0xFFu) : (int)pb;
          const int up = (int)((wm >> (8 * j)) & 0xFFu), down = (int)((w1 >> (8 * j)) & 0xFFu);
          tw[j] = (uint32_t)v | (((uint32_t)(right - left) & 0x1FFu) << 8) | (((uint32_t)(down - up) & 0x1FFu) << 17);
        }
        *reinterpret_cast<uint4*>(t8 + (size_t)y * w + x4) = make_uint4(tw[0], tw[1], tw[2], tw[3]);
      }
    }
    if (kTex) wm = w0;
    w0 = w1;
    n0 = n1;
  }
}

// Quad image of a u8 frame only (stateless interpolation entry point).
__global__ void build_quad_kernel(const uint8_t* __restrict__ src, uint32_t* __restrict__ dst, int w, int h) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  if (x >= w) return;
  const int x1 = min(x + 1, w - 1);
  const int y1 = min(y + 1, h - 1);
  const uint8_t* r0 = src + (size_t)y * w;
  const uint8_t* r1 = src + (size_t)y1 * w;
  dst[(size_t)y * w + x] = (uint32_t)r0[x] | ((uint32_t)r0[x1] << 8) | ((uint32_t)r1[x] << 16) |
                           ((uint32_t)r1[x1] << 24);
}

// sample() (flow.cpp:45-57) through a quad image: one 16-byte gather.
__device__ __forceinline__ float sample_quadf(const float4* __restrict__ q, int w, int h, float x, float y) {
  x = clamp_ref(x, 0.0f, (float)(w - 1));
  y = clamp_ref(y, 0.0f, (float)(h - 1));
  const int x0 = (int)x;
  const int y0 = (int)y;
  const float fx = fsub(x, (float)x0);
  const float fy = fsub(y, (float)y0);
  const float4 a = __ldg(q + (size_t)y0 * w + x0);
  const float top = lerp_ref(a.x, a.y, fx);
  const float bot = lerp_ref(a.z, a.w, fx);
  return lerp_ref(top, bot, fy);
}

// ---------------------------------------------------------------- dense LK

// Bilinear densification of the patch grid at one pixel: solve_level's
// output loop, flow.cpp:224-245.
__device__ __forceinline__ void densify_at(const GridGeom& g, int x, int y, float& u, float& v) {
  const int j = __ldg(g.iy + y);
  const float fy = __ldg(g.wy + y);
  const int i = __ldg(g.ix + x);
  const float fx = __ldg(g.wx + x);
  const int i0 = min(i, g.ncx - 1), i1 = min(i + 1, g.ncx - 1);
  const int j0 = min(j, g.ncy - 1), j1 = min(j + 1, g.ncy - 1);
  const size_t r0 = (size_t)j0 * g.ncx, r1 = (size_t)j1 * g.ncx;
  const float u00 = __ldg(g.pu + r0 + i0), u10 = __ldg(g.pu + r0 + i1);
  const float u01 = __ldg(g.pu + r1 + i0), u11 = __ldg(g.pu + r1 + i1);
  const float v00 = __ldg(g.pv + r0 + i0), v10 = __ldg(g.pv + r0 + i1);
  const float v01 = __ldg(g.pv + r1 + i0), v11 = __ldg(g.pv + r1 + i1);
  const float u_top = lerp_ref(u00, u10, fx), u_bot = lerp_ref(u01, u11, fx);
  const float v_top = lerp_ref(v00, v10, fx), v_bot = lerp_ref(v01, v11, fx);
  u = lerp_ref(u_top, u_bot, fy);
  v = lerp_ref(v_top, v_bot, fy);
}

// upsample_flow evaluated at one fine pixel (flow.cpp:130-147): bilinear
// sample of the densified coarse field, divided by the level ratio.  Only
// the values at the patch centres are ever read by solve_level (:174-175).
__device__ __forceinline__ void upsample_at(const GridGeom& c, int fw, int fh, int x, int y, float& u,
                                            float& v) {
  const float rx = __fdiv_rn((float)c.w, (float)fw);
  const float ry = __fdiv_rn((float)c.h, (float)fh);
  const float sy = fsub(fmul(fadd((float)y, 0.5f), ry), 0.5f);
  const float sx = fsub(fmul(fadd((float)x, 0.5f), rx), 0.5f);
  const Tap t = make_tap(sx, sy, c.w, c.h);
  float u00, v00, u10, v10, u01, v01, u11, v11;
  densify_at(c, t.x0, t.y0, u00, v00);
  densify_at(c, t.x1, t.y0, u10, v10);
  densify_at(c, t.x0, t.y1, u01, v01);
  densify_at(c, t.x1, t.y1, u11, v11);
  const float us = lerp_ref(lerp_ref(u00, u10, t.fx), lerp_ref(u01, u11, t.fx), t.fy);
  const float vs = lerp_ref(lerp_ref(v00, v10, t.fx), lerp_ref(v01, v11, t.fx), t.fy);
  u = __fdiv_rn(us, rx);
  v = __fdiv_rn(vs, ry);
}

// Central-difference gradients with replicate padding, flow.cpp:60-73.
__device__ __forceinline__ float grad_x(const float* __restrict__ im, int w, int x, int y) {
  const float* r = im + (size_t)y * w;
  return fmul(0.5f, fsub(__ldg(r + min(x + 1, w - 1)), __ldg(r + max(x - 1, 0))));
}
__device__ __forceinline__ float grad_y(const float* __restrict__ im, int w, int h, int x, int y) {
  return fmul(0.5f, fsub(__ldg(im + (size_t)min(y + 1, h - 1) * w + x), __ldg(im + (size_t)max(y - 1, 0) * w + x)));
}

constexpr int kLKTileX = 8, kLKTileY = 4;  // 32 patches per block
constexpr int kLKPatches = kLKTileX * kLKTileY;
constexpr int kLKThreads = 128;

// Shared-memory footprint of one tile (floats): the prev level over the
// tile's template region + 1-pixel halo (replicate-clamped), the gradients
// (gx, gy) of the template region, and the residual products of one
// iteration (two per template pixel per patch).
__host__ __device__ inline int lk_region_w(int r) { return (kLKTileX - 1) * r + 2 * r + 3; }
__host__ __device__ inline int lk_region_h(int r) { return (kLKTileY - 1) * r + 2 * r + 3; }
__host__ __device__ inline int lk_grad_offset(int r) { return (lk_region_w(r) * lk_region_h(r) + 3) & ~3; }
__host__ __device__ inline int lk_prod_offset(int r) {
  return lk_grad_offset(r) + 2 * (lk_region_w(r) - 2) * (lk_region_h(r) - 2);
}
size_t dense_lk_smem(int r) {
  const int d = 2 * r + 1;
  return (size_t)(lk_prod_offset(r) + 2 * kLKPatches * d * d) * sizeof(float);
}

// solve_level's per-patch loop (flow.cpp:170-215) for a tile of 8x4 patches.
// The template (prev values + central-difference gradients) is staged in
// shared memory once per tile.  Each LK iteration runs in two phases:
//   A. all 128 threads compute the float products gx*residual, gy*residual
//      of every (patch, template pixel) — the residual's bilinear sample of
//      curr is one 16-byte quad gather — into shared memory;
//   B. one thread per (patch, sum) accumulates them into the fp64 sum in the
//      reference's k order (the only sequential part), then the 2x2 solve.
// The template sums gxx/gxy/gyy are exact in fp64 for every supported level
// and radius (all terms are multiples of 2^-(4l+2), the total stays below
// 2^53 of those quanta), so they are split across threads.
template <int kR>
__global__ void __launch_bounds__(kLKThreads) dense_lk_tile_kernel(DenseLKParams p) {
  extern __shared__ __align__(16) float smem[];
  const int z = blockIdx.z;  // frame pair
  GridGeom g = p.g;
  g.pu += z * g.pair_stride;
  g.pv += z * g.pair_stride;
  GridGeom coarse = p.coarse;
  coarse.pu += z * coarse.pair_stride;
  coarse.pv += z * coarse.pair_stride;
  const float* __restrict__ prev = p.prev.at((p.r0 + z) % p.R);
  const float4* __restrict__ qcurr = p.qcurr.at((p.r0 + z + 1) % p.R);
  __shared__ float s_u[kLKPatches], s_v[kLKPatches];
  __shared__ int s_cx[kLKPatches], s_cy[kLKPatches], s_solve[kLKPatches];
  __shared__ double s_part[3][4][kLKPatches];
  __shared__ double s_gxx[kLKPatches], s_gxy[kLKPatches], s_gyy[kLKPatches], s_inv[kLKPatches];
  __shared__ double s_b[2][kLKPatches];
  const int r = kR > 0 ? kR : p.radius;
  const int D = 2 * r + 1, P2 = D * D;
  const int w = g.w, h = g.h;
  const int t = threadIdx.x;
  const int i0 = blockIdx.x * kLKTileX, j0 = p.jt0 + blockIdx.y * kLKTileY;
  const int i1 = min(i0 + kLKTileX, g.ncx) - 1, j1 = min(j0 + kLKTileY, g.ncy) - 1;
  const int rx0 = __ldg(g.cx + i0) - r - 1, ry0 = __ldg(g.cy + j0) - r - 1;
  const int rw = __ldg(g.cx + i1) - __ldg(g.cx + i0) + 2 * r + 3;
  const int rh = __ldg(g.cy + j1) - __ldg(g.cy + j0) + 2 * r + 3;
  const int pitch = lk_region_w(r), gpitch = pitch - 2;
  float* sP = smem;                                                   // [rh][pitch]
  float2* sG = reinterpret_cast<float2*>(smem + lk_grad_offset(r));   // [rh-2][gpitch]
  float* sB1 = smem + lk_prod_offset(r);                              // [patch][P2]
  float* sB2 = sB1 + kLKPatches * P2;

#pragma unroll 4
  for (int e = t; e < rw * rh; e += kLKThreads) {
    const int yy = e / rw, xx = e - yy * rw;
    const int sy = clampi(ry0 + yy, 0, h - 1), sx = clampi(rx0 + xx, 0, w - 1);
    sP[yy * pitch + xx] = __ldg(prev + (size_t)sy * w + sx);
  }
  if (t < kLKPatches) {
    const int i = i0 + t % kLKTileX, j = j0 + t / kLKTileX;
    const bool valid = i < g.ncx && j < g.ncy;
    const int cx = __ldg(g.cx + (valid ? i : i0)), cy = __ldg(g.cy + (valid ? j : j0));
    float u = 0.0f, v = 0.0f;
    if (valid && p.has_coarse) upsample_at(coarse, w, h, cx, cy, u, v);
    s_cx[t] = cx;
    s_cy[t] = cy;
    s_u[t] = u;
    s_v[t] = v;
    s_solve[t] = valid;
  }
  __syncthreads();
  // gradients at every template position (flow.cpp:60-73: the clamped
  // neighbours are reproduced by the replicate-staged halo)
  for (int e = t; e < (rw - 2) * (rh - 2); e += kLKThreads) {
    const int yy = e / (rw - 2) + 1, xx = e - (yy - 1) * (rw - 2) + 1;
    const float* row = sP + yy * pitch;
    sG[(yy - 1) * gpitch + (xx - 1)] =
        make_float2(fmul(0.5f, fsub(row[xx + 1], row[xx - 1])), fmul(0.5f, fsub(row[pitch + xx], row[xx - pitch])));
  }
  __syncthreads();
  // template sums (flow.cpp:177-194): 4 row-parts per patch, exact
  {
    const int pt = t % kLKPatches, part = t / kLKPatches;
    const int cx = s_cx[pt], cy = s_cy[pt];
    double gxx = 0.0, gxy = 0.0, gyy = 0.0;
    for (int oy = -r + part; oy <= r; oy += 4) {
      const int py = clampi(cy + oy, 0, h - 1);
      const float2* grow = sG + (py - ry0 - 1) * gpitch - rx0 - 1;
      for (int ox = -r; ox <= r; ++ox) {
        const float2 gr = grow[clampi(cx + ox, 0, w - 1)];
        gxx = dadd(gxx, (double)fmul(gr.x, gr.x));
        gxy = dadd(gxy, (double)fmul(gr.x, gr.y));
        gyy = dadd(gyy, (double)fmul(gr.y, gr.y));
      }
    }
    s_part[0][part][pt] = gxx;
    s_part[1][part][pt] = gxy;
    s_part[2][part][pt] = gyy;
  }
  __syncthreads();
  if (t < kLKPatches) {
    const double gxx = dadd(dadd(dadd(s_part[0][0][t], s_part[0][1][t]), s_part[0][2][t]), s_part[0][3][t]);
    const double gxy = dadd(dadd(dadd(s_part[1][0][t], s_part[1][1][t]), s_part[1][2][t]), s_part[1][3][t]);
    const double gyy = dadd(dadd(dadd(s_part[2][0][t], s_part[2][1][t]), s_part[2][2][t]), s_part[2][3][t]);
    const bool solve = s_solve[t] && min_eigenvalue(gxx, gxy, gyy) > dmul(1e-4, (double)P2);
    s_solve[t] = solve ? 1 : (s_solve[t] ? 2 : 0);  // 1 solve, 2 valid-but-flat, 0 padding
    s_gxx[t] = gxx;
    s_gxy[t] = gxy;
    s_gyy[t] = gyy;
    if (solve) s_inv[t] = __ddiv_rn(1.0, dsub(dmul(gxx, gyy), dmul(gxy, gxy)));
  }
  __syncthreads();
  const float max_step = (float)r;
  for (int it = 0; it < p.iterations; ++it) {
    // phase A: residual products (flow.cpp:202-205, float)
    // (batches of kU gathers in flight per thread)
    constexpr int kU = 6;
    for (int e0 = t; e0 < kLKPatches * P2; e0 += kLKThreads * kU) {
      float4 q[kU];
      float fxs[kU], fys[kU];
      int pxs[kU], pys[kU];
      bool ok[kU];
#pragma unroll
      for (int c = 0; c < kU; ++c) {
        const int e = e0 + c * kLKThreads;
        const int pt = e / P2, k = e - pt * P2;
        ok[c] = e < kLKPatches * P2 && s_solve[pt] == 1;
        q[c] = make_float4(0.f, 0.f, 0.f, 0.f);
        pxs[c] = pys[c] = 0;
        fxs[c] = fys[c] = 0.f;
        if (ok[c]) {
          const int oy = k / D - r, ox = k - (k / D) * D - r;
          const int px = clampi(s_cx[pt] + ox, 0, w - 1), py = clampi(s_cy[pt] + oy, 0, h - 1);
          // sample() taps (flow.cpp:45-53) of curr at (px + u, py + v); u, v
          // are finite, so FMNMX clamps and the RZ-add truncation are exact
          const float x = fminf(fmaxf(fadd((float)px, s_u[pt]), 0.0f), (float)(w - 1));
          const float y = fminf(fmaxf(fadd((float)py, s_v[pt]), 0.0f), (float)(h - 1));
          int x0, y0;
          const float x0f = trunc_magic(x, x0), y0f = trunc_magic(y, y0);
          fxs[c] = fsub(x, x0f);
          fys[c] = fsub(y, y0f);
          q[c] = __ldg(qcurr + (size_t)y0 * w + x0);
          pxs[c] = px;
          pys[c] = py;
        }
      }
#pragma unroll
      for (int c = 0; c < kU; ++c) {
        if (!ok[c]) continue;
        const int e = e0 + c * kLKThreads;
        const int px = pxs[c], py = pys[c];
        const float tval = sP[(py - ry0) * pitch + (px - rx0)];
        const float2 gr = sG[(py - ry0 - 1) * gpitch + (px - rx0 - 1)];
        const float s = lerp_ref(lerp_ref(q[c].x, q[c].y, fxs[c]), lerp_ref(q[c].z, q[c].w, fxs[c]), fys[c]);
        const float residual = fsub(s, tval);
        sB1[e] = fmul(gr.x, residual);
        sB2[e] = fmul(gr.y, residual);
      }
    }
    __syncthreads();
    // phase B: the ordered fp64 sums b1 (warp 0) and b2 (warp 1)
    if (t < 2 * kLKPatches) {
      const int pt = t % kLKPatches;
      if (s_solve[pt] == 1) {
        const float* src = (t < kLKPatches ? sB1 : sB2) + pt * P2;
        double acc = 0.0;
#pragma unroll 9
        for (int k = 0; k < P2; ++k) acc = dadd(acc, (double)src[k]);
        s_b[t / kLKPatches][pt] = acc;
      }
    }
    __syncthreads();
    if (t < kLKPatches && s_solve[t] == 1) {
      const double b1 = s_b[0][t], b2 = s_b[1][t];
      const double gxx = s_gxx[t], gxy = s_gxy[t], gyy = s_gyy[t], inv_det = s_inv[t];
      float du = __double2float_rn(dmul(-dsub(dmul(gyy, b1), dmul(gxy, b2)), inv_det));
      float dv = __double2float_rn(dmul(-dsub(dmul(gxx, b2), dmul(gxy, b1)), inv_det));
      du = clamp_ref(du, -max_step, max_step);
      dv = clamp_ref(dv, -max_step, max_step);
      s_u[t] = fadd(s_u[t], du);
      s_v[t] = fadd(s_v[t], dv);
    }
    __syncthreads();
  }
  if (t < kLKPatches && s_solve[t] != 0) {
    const int i = i0 + t % kLKTileX, j = j0 + t / kLKTileX;
    g.pu[(size_t)j * g.ncx + i] = s_u[t];
    g.pv[(size_t)j * g.ncx + i] = s_v[t];
  }
}

// ---------------------------------------------------------------- dense LK, warp form
// The tile of 8x4 patches for the preset radii (4, 6) when no template
// coordinate needs clamping (extent > 2r+1: patch_centers, flow.cpp:97-107,
// keeps every patch inside the level).  After staging the template region,
// each warp owns one tile row (8 patches) and runs their whole solve alone —
// only __syncwarp, no block barriers:
//  * template sums (exact in fp64) split over 4 row-parts
//    per patch and combined with xor-shuffles;
//  * per iteration, the bilinear split of every template column / row —
//    sample(curr, px + u, py + v) (flow.cpp:203) pairs a column's x-split
//    with a row's y-split — is tabulated; lanes = (row within a group of RPG
//    rows, column) of one patch compute the products gx*res, gy*res;
//  * 16 lanes (patch, b1|b2) then run the ordered fp64 sums in the
//    reference's k order (flow.cpp:204-205) and every lane applies its
//    patch's 2x2 solve (flow.cpp:207-213).
__host__ __device__ constexpr int lk_pick_pitch(int rw, int d, int rpg) {
  // smallest pitch >= rw whose RPG rows of D columns fall in distinct banks
  for (int p = rw; p < rw + 32; ++p) {
    bool ok = true;
    for (int a = 1; a < rpg; ++a) {
      const int m = (a * p) % 32;
      if (m < d || m > 32 - d) ok = false;
    }
    if (ok) return p;
  }
  return rw;
}

template <int kR>
struct LKWarp {
  static constexpr int D = 2 * kR + 1, P2 = D * D;
  static constexpr int RPG = 32 / D;                // template rows per lane group
  static constexpr int NG = (D + RPG - 1) / RPG;    // lane groups per patch
  static constexpr int kPW = kLKTileX;              // patches per warp (one tile row)
  static constexpr int rw = (kLKTileX - 1) * kR + 2 * kR + 3;
  static constexpr int rows = (kLKTileY - 1) * kR + 2 * kR + 3;
  static constexpr int pitch = lk_pick_pitch(rw, D, RPG);
  static constexpr int plane = (pitch * rows + 3) & ~3;                   // floats
  // products of one lane group: two planes (gx*res, gy*res) of [kPW][S]
  // floats per warp; S even and S, the plane offset PO chosen so that the 16
  // phase-B lanes' 8-byte reads hit distinct bank pairs where possible
  static constexpr int S = ((RPG * D + 1) & ~1) + (((((RPG * D + 1) & ~1) / 2) % 2) ? 0 : 2);
  static constexpr int PO = kPW * S + ((kPW * S) % 32 == 16 ? 0 : (48 - (kPW * S) % 32) % 32);
  static constexpr int b_off = 3 * plane;                                 // float [warp][2][PO]
  static constexpr int t_off = b_off + kLKTileY * 2 * PO;                 // float2 [warp][2][kPW][D]
  static constexpr int floats = t_off + 2 * kLKTileY * 2 * kPW * D;
};
static_assert(kLKThreads == 32 * kLKTileY, "one warp per tile row");

template <int kR, bool kU8>
__global__ void __launch_bounds__(kLKThreads) dense_lk_warp_kernel(DenseLKParams p) {
  using G = LKWarp<kR>;
  constexpr int D = G::D, P2 = G::P2, RPG = G::RPG, NG = G::NG, kPW = G::kPW, pitch = G::pitch;
  extern __shared__ __align__(16) float smem[];
  const int z = blockIdx.z;  // frame pair
  GridGeom g = p.g;
  g.pu += z * g.pair_stride;
  g.pv += z * g.pair_stride;
  GridGeom coarse = p.coarse;
  coarse.pu += z * coarse.pair_stride;
  coarse.pv += z * coarse.pair_stride;
  // kU8 (level 0 of the dense path): prev = the u8 frame, curr = its u8 quad
  // image — exactly the values to_float / the float quad would hold
  const float* __restrict__ prev = kU8 ? nullptr : p.prev.at((p.r0 + z) % p.R);
  const float4* __restrict__ qcurr = kU8 ? nullptr : p.qcurr.at((p.r0 + z + 1) % p.R);
  const uint8_t* __restrict__ prev8 = kU8 ? p.prev8.at((p.r0 + z) % p.R) : nullptr;
  const uint32_t* __restrict__ qcurr8 = kU8 ? p.qcurr8.at((p.r0 + z + 1) % p.R) : nullptr;
  const int w = g.w, h = g.h;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int i0 = blockIdx.x * kLKTileX, j0 = p.jt0 + blockIdx.y * kLKTileY;
  const int i1 = min(i0 + kLKTileX, g.ncx) - 1, j1 = min(j0 + kLKTileY, g.ncy) - 1;
  const int rx0 = __ldg(g.cx + i0) - kR - 1, ry0 = __ldg(g.cy + j0) - kR - 1;
  const int rw = __ldg(g.cx + i1) - __ldg(g.cx + i0) + 2 * kR + 3;
  const int rh = __ldg(g.cy + j1) - __ldg(g.cy + j0) + 2 * kR + 3;
  float* sP = smem;               // [rows][pitch] prev, replicate-staged
  float* sGx = smem + G::plane;   // [rows][pitch] central differences
  float* sGy = smem + 2 * G::plane;
  float* sB = smem + G::b_off + warp * (2 * G::PO);  // [2][PO]: plane b1 at 0, plane b2 at PO
  float2* sX = reinterpret_cast<float2*>(smem + G::t_off) + warp * (2 * kPW * D);  // [kPW][D] (x0, fx)
  float2* sY = sX + kPW * D;                                                        // [kPW][D] (y0*w, fy)

  // u8 interior regions (no replicate clamp) of 4-byte aligned rows: aligned
  // words, four taps each
  const bool words = kU8 && (w & 3) == 0 && ((uintptr_t)prev8 & 3) == 0 && rx0 >= 0 && ry0 >= 0 &&
                     rx0 + rw <= w && ry0 + rh <= h;
  if (words) {
    const int a0 = rx0 & ~3, nw = (rx0 + rw - a0 + 3) >> 2;
    const uint32_t* src = reinterpret_cast<const uint32_t*>(prev8 + (size_t)ry0 * w + a0);
    const int wpr = w >> 2;
    for (int e = t; e < rh * nw; e += kLKThreads) {
      const int yy = e / nw, wd = e - yy * nw;
      const uint32_t q = __ldg(src + yy * wpr + wd);
      const int xx = a0 - rx0 + 4 * wd;  // region column of byte 0 (>= -3)
      float* dst = sP + yy * pitch + xx;
#pragma unroll
      for (int b = 0; b < 4; ++b)
        if (xx + b >= 0 && xx + b < rw) dst[b] = __fsub_rn(__uint_as_float(__byte_perm(q, 0x4B000000u, 0x7540 + b)),
                                                          8388608.0f);
    }
  } else if (!kU8 && (w & 3) == 0 && ((uintptr_t)prev & 15) == 0 && rx0 >= 0 && ry0 >= 0 && rx0 + rw <= w &&
             ry0 + rh <= h) {
    // fp32 interior regions: aligned float4 loads
    const int a0 = rx0 & ~3, nw = (rx0 + rw - a0 + 3) >> 2;
    const float4* src = reinterpret_cast<const float4*>(prev + (size_t)ry0 * w + a0);
    const int wpr = w >> 2;
    for (int e = t; e < rh * nw; e += kLKThreads) {
      const int yy = e / nw, wd = e - yy * nw;
      const float4 q = __ldg(src + yy * wpr + wd);
      const int xx = a0 - rx0 + 4 * wd;
      float* dst = sP + yy * pitch + xx;
      if (xx >= 0) dst[0] = q.x;
      if (xx + 1 >= 0 && xx + 1 < rw) dst[1] = q.y;
      if (xx + 2 >= 0 && xx + 2 < rw) dst[2] = q.z;
      if (xx + 3 < rw) dst[3] = q.w;
    }
  } else {
    for (int yy = warp; yy < rh; yy += kLKTileY) {
      const size_t roff = (size_t)clampi(ry0 + yy, 0, h - 1) * w;
      for (int xx = lane; xx < rw; xx += 32) {
        const int sx = clampi(rx0 + xx, 0, w - 1);
        sP[yy * pitch + xx] = kU8 ? u8f(__ldg(prev8 + roff + sx)) : __ldg(prev + roff + sx);
      }
    }
  }
  // this lane's patch: pl = lane & 7 of tile row `warp` (all four 8-lane parts agree)
  const int pl = lane & 7, part = lane >> 3;
  const int pi = i0 + pl, pj = j0 + warp;
  const bool valid = pi < g.ncx && pj < g.ncy;
  const int cx = __ldg(g.cx + (valid ? pi : i0)), cy = __ldg(g.cy + (valid ? pj : j0));
  float u = 0.0f, v = 0.0f;
  if (valid && p.has_coarse && part == 0) upsample_at(coarse, w, h, cx, cy, u, v);
  u = __shfl_sync(kFull, u, pl);
  v = __shfl_sync(kFull, v, pl);
  __syncthreads();
  for (int yy = 1 + warp; yy < rh - 1; yy += kLKTileY) {
    const float* row = sP + yy * pitch;
    for (int xx = 1 + lane; xx < rw - 1; xx += 32) {
      sGx[yy * pitch + xx] = fmul(0.5f, fsub(row[xx + 1], row[xx - 1]));
      sGy[yy * pitch + xx] = fmul(0.5f, fsub(row[pitch + xx], row[xx - pitch]));
    }
  }
  __syncthreads();
  // template sums (flow.cpp:177-194), rows part, part+4, ... of patch pl
  const int tb = (cy - ry0) * pitch + (cx - rx0);  // region offset of the patch centre
  double gxx = 0.0, gxy = 0.0, gyy = 0.0;
  for (int oy = -kR + part; oy <= kR; oy += 4) {
#pragma unroll
    for (int ox = -kR; ox <= kR; ++ox) {
      const int o = tb + oy * pitch + ox;
      const float a = sGx[o], b = sGy[o];
      gxx = dadd(gxx, (double)fmul(a, a));
      gxy = dadd(gxy, (double)fmul(a, b));
      gyy = dadd(gyy, (double)fmul(b, b));
    }
  }
#pragma unroll
  for (int m = 8; m <= 16; m <<= 1) {  // exact, so any combination order
    gxx = dadd(gxx, __shfl_xor_sync(kFull, gxx, m));
    gxy = dadd(gxy, __shfl_xor_sync(kFull, gxy, m));
    gyy = dadd(gyy, __shfl_xor_sync(kFull, gyy, m));
  }
  const bool solve = valid && min_eigenvalue(gxx, gxy, gyy) > dmul(1e-4, (double)P2);
  const double inv_det = solve ? __ddiv_rn(1.0, dsub(dmul(gxx, gyy), dmul(gxy, gxy))) : 0.0;
  const unsigned solved = __ballot_sync(kFull, solve) & 0xFFu;  // bit j: patch j of this warp
  const float max_step = (float)kR;
  const float wm = (float)(w - 1), hm = (float)(h - 1);
  // the lane's place in a patch: template row ry of each group, column ox
  const int ry = lane / D, ox = lane - (lane / D) * D;
  const bool lane_on = lane < RPG * D;
  const int oxs = lane_on ? ox : 0;
  uint32_t tbj[kPW];  // region byte offsets of the warp's patch centres
#pragma unroll
  for (int j = 0; j < kPW; ++j) tbj[j] = 4u * (uint32_t)__shfl_sync(kFull, tb, j);
  // pinned: the shared window address of sP, the quad image, the 2^23 byte bias
  const uint32_t s_addr = pin((uint32_t)__cvta_generic_to_shared(sP));
  const float4* __restrict__ qcurr_p = kU8 ? nullptr : pin(qcurr);
  const uint32_t* __restrict__ qcurr8_p = kU8 ? pin(qcurr8) : nullptr;
  const uint32_t kMagic = pin(0x4B000000u);
  for (int it = 0; it < p.iterations && solved; ++it) {
    // split tables for the warp's 8 patches (flow.cpp:45-53 on px + u, py + v; u, v finite)
#pragma unroll
    for (int e0 = 0; e0 < kPW * D; e0 += 32) {
      const int e = e0 + lane;
      const int ptx = e < kPW * D ? e / D : 0, i = e - ptx * D;
      const float uj = __shfl_sync(kFull, u, ptx), vj = __shfl_sync(kFull, v, ptx);
      const int cxj = __shfl_sync(kFull, cx, ptx), cyj = __shfl_sync(kFull, cy, ptx);
      if (e < kPW * D) {
        const float x = fminf(fmaxf(fadd((float)(cxj + i - kR), uj), 0.0f), wm);
        const float y = fminf(fmaxf(fadd((float)(cyj + i - kR), vj), 0.0f), hm);
        int x0, y0;
        const float x0f = trunc_magic(x, x0), y0f = trunc_magic(y, y0);
        sX[e] = make_float2(__int_as_float(x0), fsub(x, x0f));
        sY[e] = make_float2(__int_as_float(y0 * w), fsub(y, y0f));
      }
    }
    __syncwarp();
    // lane group by lane group (template rows gg*RPG .. gg*RPG+RPG-1, i.e. k
    // = gg*RPG*D + lane): residual products gx*res, gy*res of the warp's 8
    // patches (flow.cpp:202-205), then 16 lanes = (patch, b1|b2) extend the
    // ordered fp64 sums by those k (flow.cpp:204-205, k order kept)
    // the lane's column split of each patch is the same for every lane group
    float fxj[kPW];
    int xj[kPW];
#pragma unroll
    for (int j = 0; j < kPW; ++j) {
      const float2 X = sX[j * D + oxs];
      fxj[j] = X.y;
      xj[j] = __float_as_int(X.x);
    }
    double acc = 0.0;
#pragma unroll 1
    for (int gg = 0; gg < NG; ++gg) {
      const int oy = gg * RPG + ry;
      const bool on = lane_on && oy < D;
      const int oyc = oy < D ? oy : 0;  // lanes off the template compute in bounds, store nothing
      const uint32_t aoff = s_addr + 4u * (uint32_t)((oyc - kR) * pitch + (oxs - kR));
      constexpr int kJB = 4;  // patches per gather batch
#pragma unroll
      for (int jb = 0; jb < kPW; jb += kJB) {
        if (!((solved >> jb) & ((1u << kJB) - 1u))) continue;  // warp-uniform
        float4 q[kJB];
        uint32_t q8[kJB];
        float fy[kJB];
#pragma unroll
        for (int jj = 0; jj < kJB; ++jj) {
          const float2 Y = sY[(jb + jj) * D + oyc];
          fy[jj] = Y.y;
          const int qi = __float_as_int(Y.x) + xj[jb + jj];
          if (kU8) q8[jj] = __ldg(qcurr8_p + qi);
          else q[jj] = __ldg(qcurr_p + qi);
        }
#pragma unroll
        for (int jj = 0; jj < kJB; ++jj) {
          const int j = jb + jj;
          if (!((solved >> j) & 1u)) continue;  // warp-uniform
          const uint32_t ao = aoff + tbj[j];
          const float fx = fxj[j];
          float smp;
          if (kU8) {
            // the u8 quad as two fp32x2 pairs (a00, a01), (a10, a11): 2^23 + b
            // via PRMT; b - a of biased taps is exact, f*(b-a) one FMUL2, the
            // adds scalar (sample(), flow.cpp:54-56, rounding by rounding)
            const uint32_t v = q8[jj];
            const f32x2 B0 = pk2(__uint_as_float(__byte_perm(v, kMagic, 0x7540)),
                                 __uint_as_float(__byte_perm(v, kMagic, 0x7542)));
            const f32x2 B1 = pk2(__uint_as_float(__byte_perm(v, kMagic, 0x7541)),
                                 __uint_as_float(__byte_perm(v, kMagic, 0x7543)));
            const f32x2 A = sub2(B0, pk2(8388608.0f, 8388608.0f));
            const f32x2 M = mul2(pk2(fx, fx), sub2(B1, B0));
            smp = lerp_ref(__fadd_rn(lo2(A), lo2(M)), __fadd_rn(hi2(A), hi2(M)), fy[jj]);
          } else {
            const float4 a = q[jj];
            smp = lerp_ref(lerp_ref(a.x, a.y, fx), lerp_ref(a.z, a.w, fx), fy[jj]);
          }
          const float res = fsub(smp, lds_f32<0>(ao));
          const float b1 = fmul(lds_f32<4 * G::plane>(ao), res), b2 = fmul(lds_f32<8 * G::plane>(ao), res);
          if (on) {
            sB[j * G::S + lane] = b1;
            sB[G::PO + j * G::S + lane] = b2;
          }
        }
      }
      __syncwarp();
      if (lane < 2 * kPW && ((solved >> pl) & 1u)) {
        const int nk = min(RPG, D - gg * RPG) * D;
        const float* src = sB + (lane >> 3) * G::PO + pl * G::S;
        const float2* src2 = reinterpret_cast<const float2*>(src);
#pragma unroll 7
        for (int m = 0; m < nk / 2; ++m) {
          const float2 f = src2[m];
          acc = dadd(acc, (double)f.x);
          acc = dadd(acc, (double)f.y);
        }
        if (nk & 1) acc = dadd(acc, (double)src[nk - 1]);
      }
      __syncwarp();
    }
    const double b1 = __shfl_sync(kFull, acc, pl), b2 = __shfl_sync(kFull, acc, pl + 8);
    if (solve) {
      float du = __double2float_rn(dmul(-dsub(dmul(gyy, b1), dmul(gxy, b2)), inv_det));
      float dv = __double2float_rn(dmul(-dsub(dmul(gxx, b2), dmul(gxy, b1)), inv_det));
      du = clamp_ref(du, -max_step, max_step);
      dv = clamp_ref(dv, -max_step, max_step);
      u = fadd(u, du);
      v = fadd(v, dv);
    }
  }
  if (lane < kPW && valid) {
    EVSIM_CHECK(pi >= 0 && pi < g.ncx && pj >= 0 && pj < g.ncy, "LK patch-grid store");
    g.pu[(size_t)pj * g.ncx + pi] = u;
    g.pv[(size_t)pj * g.ncx + pi] = v;
  }
}

// Fallback for radii whose tile does not fit in shared memory (r > 10): one
// thread per patch, template and gradients straight from L1/L2.
__global__ void __launch_bounds__(128) dense_lk_global_kernel(DenseLKParams p) {
  const int pid = blockIdx.x * blockDim.x + threadIdx.x;
  const int z = blockIdx.y;  // frame pair
  GridGeom g = p.g;
  g.pu += z * g.pair_stride;
  g.pv += z * g.pair_stride;
  GridGeom coarse = p.coarse;
  coarse.pu += z * coarse.pair_stride;
  coarse.pv += z * coarse.pair_stride;
  const float* __restrict__ prev = p.prev.at((p.r0 + z) % p.R);
  const float4* __restrict__ qcurr = p.qcurr.at((p.r0 + z + 1) % p.R);
  if (pid >= g.ncx * (p.jt1 - p.jt0)) return;
  const int i = pid % g.ncx;
  const int j = p.jt0 + pid / g.ncx;
  const int cx = __ldg(g.cx + i);
  const int cy = __ldg(g.cy + j);
  const int w = g.w, h = g.h, r = p.radius;
  float u = 0.0f, v = 0.0f;
  if (p.has_coarse) upsample_at(coarse, w, h, cx, cy, u, v);
  double gxx = 0.0, gxy = 0.0, gyy = 0.0;
  for (int oy = -r; oy <= r; ++oy) {
    const int py = clampi(cy + oy, 0, h - 1);
    for (int ox = -r; ox <= r; ++ox) {
      const int px = clampi(cx + ox, 0, w - 1);
      const float a = grad_x(prev, w, px, py);
      const float b = grad_y(prev, w, h, px, py);
      gxx = dadd(gxx, (double)fmul(a, a));
      gxy = dadd(gxy, (double)fmul(a, b));
      gyy = dadd(gyy, (double)fmul(b, b));
    }
  }
  const int patch_pixels = (2 * r + 1) * (2 * r + 1);
  if (min_eigenvalue(gxx, gxy, gyy) > dmul(1e-4, (double)patch_pixels)) {
    const double inv_det = __ddiv_rn(1.0, dsub(dmul(gxx, gyy), dmul(gxy, gxy)));
    const float max_step = (float)r;
    for (int it = 0; it < p.iterations; ++it) {
      double b1 = 0.0, b2 = 0.0;
      for (int oy = -r; oy <= r; ++oy) {
        const int py = clampi(cy + oy, 0, h - 1);
        const float syv = fadd((float)py, v);
        for (int ox = -r; ox <= r; ++ox) {
          const int px = clampi(cx + ox, 0, w - 1);
          const float a = grad_x(prev, w, px, py);
          const float b = grad_y(prev, w, h, px, py);
          const float tval = __ldg(prev + (size_t)py * w + px);
          const float residual = fsub(sample_quadf(qcurr, w, h, fadd((float)px, u), syv), tval);
          b1 = dadd(b1, (double)fmul(a, residual));
          b2 = dadd(b2, (double)fmul(b, residual));
        }
      }
      float du = __double2float_rn(dmul(-dsub(dmul(gyy, b1), dmul(gxy, b2)), inv_det));
      float dv = __double2float_rn(dmul(-dsub(dmul(gxx, b2), dmul(gxy, b1)), inv_det));
      du = clamp_ref(du, -max_step, max_step);
      dv = clamp_ref(dv, -max_step, max_step);
      u = fadd(u, du);
      v = fadd(v, dv);
    }
  }
  g.pu[(size_t)j * g.ncx + i] = u;
  g.pv[(size_t)j * g.ncx + i] = v;
}

__global__ void densify_kernel(GridGeom g, float* __restrict__ du, float* __restrict__ dv) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  if (x >= g.w) return;
  float u, v;
  densify_at(g, x, y, u, v);
  du[(size_t)y * g.w + x] = u;
  dv[(size_t)y * g.w + x] = v;
}

// ---------------------------------------------------------------- sparse LK

// sample() of the materialised gradient images and of P (flow.cpp:328-334)
// through the template texels: the four taps carry (value, gx, gy), so one
// bilinear sample of all three is four 16-byte loads (one when the position
// is integral: lerp(a, b, 0) = a exactly).
__device__ __forceinline__ void sample_texel(const float4* __restrict__ tex, int w, int h, float sx, float sy,
                                             float& a, float& b, float& val) {
  const Tap t = make_tap(sx, sy, w, h);
  const float4* r0 = tex + (size_t)t.y0 * w;
  const float4 q00 = __ldg(r0 + t.x0);
  if (t.fx == 0.0f && t.fy == 0.0f) {
    val = q00.x;
    a = q00.y;
    b = q00.z;
    return;
  }
  const float4* r1 = tex + (size_t)t.y1 * w;
  const float4 q10 = __ldg(r0 + t.x1), q01 = __ldg(r1 + t.x0), q11 = __ldg(r1 + t.x1);
  a = lerp_ref(lerp_ref(q00.y, q10.y, t.fx), lerp_ref(q01.y, q11.y, t.fx), t.fy);
  b = lerp_ref(lerp_ref(q00.z, q10.z, t.fx), lerp_ref(q01.z, q11.z, t.fx), t.fy);
  val = lerp_ref(lerp_ref(q00.x, q10.x, t.fx), lerp_ref(q01.x, q11.x, t.fx), t.fy);
}

// Level 0 from u8 data: template positions are integral there (px = x:
// the level ratio is 1), so sample() of the gradient images and of P is one
// tap (lerp(a, b, 0) = a) — the packed texel; the residual's sample of curr
// reads the u8 quad (bytes convert to the fp32 level values exactly).
__device__ __forceinline__ void sample_texel8(const uint32_t* __restrict__ t8, int w, int h, float sx, float sy,
                                              float& a, float& b, float& val) {
  const int x = (int)clamp_ref(sx, 0.0f, (float)(w - 1));
  const int y = (int)clamp_ref(sy, 0.0f, (float)(h - 1));
  const uint32_t t = __ldg(t8 + (size_t)y * w + x);
  val = (float)(t & 0xFFu);
  a = fmul(0.5f, (float)((int)(t << 15) >> 23));
  b = fmul(0.5f, (float)((int)(t << 6) >> 23));
}

__device__ __forceinline__ float sample_quad8(const uint32_t* __restrict__ q, int w, int h, float x, float y) {
  x = clamp_ref(x, 0.0f, (float)(w - 1));
  y = clamp_ref(y, 0.0f, (float)(h - 1));
  const int x0 = (int)x;
  const int y0 = (int)y;
  const float fx = fsub(x, (float)x0);
  const float fy = fsub(y, (float)y0);
  const uint32_t a = __ldg(q + (size_t)y0 * w + x0);
  const float top = lerp_ref((float)(a & 0xFFu), (float)((a >> 8) & 0xFFu), fx);
  const float bot = lerp_ref((float)((a >> 16) & 0xFFu), (float)(a >> 24), fx);
  return lerp_ref(top, bot, fy);
}

// estimate_sparse_flow's per-point loop (flow.cpp:309-380), one thread per point.
__global__ void __launch_bounds__(128, 7) sparse_lk_kernel(SparseLKParams p) {
  const int z = blockIdx.y;  // frame pair
  const int64_t M = p.n_points ? (int64_t)p.n_points[z] : p.n_points_host;
  const uint32_t* points = p.points + z * p.pair_stride;
  float2* disp = p.disp + z * p.pair_stride;
  uint8_t* status = p.status + z * p.pair_stride;
  const int sp = (p.r0 + z) % p.R, sc = (p.r0 + z + 1) % p.R;
  const int r = p.radius;
  const int patch_pixels = (2 * r + 1) * (2 * r + 1);
  const float max_step = (float)r;
  const float diverge_limit = fmul(2.0f, (float)max(p.w0, p.h0));
  const float w0 = (float)p.w0, h0 = (float)p.h0;
  for (int64_t pi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pi < M;
       pi += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t idx = points[pi];
    const int ptx = (int)(idx % (uint32_t)p.w0);
    const int pty = (int)(idx / (uint32_t)p.w0);
    float u = 0.0f, v = 0.0f;
    bool lost = false, solved_any = false;
    for (int l = p.levels - 1; l >= 0 && !lost; --l) {
      const int w = p.dims[l].w, h = p.dims[l].h;
      const bool u8l = l == 0 && p.u8_level0;
      const float4* T = u8l ? nullptr : p.tex[l].at(sp);
      const float4* C = u8l ? nullptr : p.qcurr[l].at(sc);
      const uint32_t* T8 = u8l ? p.tex8.at(sp) : nullptr;
      const uint32_t* C8 = u8l ? p.qcurr8.at(sc) : nullptr;
      const float px = fsub(fmul(fadd((float)ptx, 0.5f), __fdiv_rn((float)w, w0)), 0.5f);
      const float py = fsub(fmul(fadd((float)pty, 0.5f), __fdiv_rn((float)h, h0)), 0.5f);
      if (l != p.levels - 1) {
        u = fmul(u, __fdiv_rn((float)w, (float)p.dims[l + 1].w));
        v = fmul(v, __fdiv_rn((float)h, (float)p.dims[l + 1].h));
      }
      double gxx = 0.0, gxy = 0.0, gyy = 0.0;
      for (int oy = -r; oy <= r; ++oy) {
        const float sy = fadd(py, (float)oy);
        for (int ox = -r; ox <= r; ++ox) {
          float a, b, tv;
          if (u8l) sample_texel8(T8, w, h, fadd(px, (float)ox), sy, a, b, tv);
          else sample_texel(T, w, h, fadd(px, (float)ox), sy, a, b, tv);
          gxx = dadd(gxx, (double)fmul(a, a));
          gxy = dadd(gxy, (double)fmul(a, b));
          gyy = dadd(gyy, (double)fmul(b, b));
        }
      }
      if (min_eigenvalue(gxx, gxy, gyy) <= dmul(1e-4, (double)patch_pixels)) continue;  // flow.cpp:340-342
      solved_any = true;
      const double inv_det = __ddiv_rn(1.0, dsub(dmul(gxx, gyy), dmul(gxy, gxy)));
      for (int it = 0; it < p.iterations; ++it) {
        double b1 = 0.0, b2 = 0.0;
        for (int oy = -r; oy <= r; ++oy) {
          const float sy = fadd(py, (float)oy);
          const float syv = fadd(sy, v);
          for (int ox = -r; ox <= r; ++ox) {
            const float sx = fadd(px, (float)ox);
            float a, b, tv;
            float smp;
            if (u8l) {
              sample_texel8(T8, w, h, sx, sy, a, b, tv);
              smp = sample_quad8(C8, w, h, fadd(sx, u), syv);
            } else {
              sample_texel(T, w, h, sx, sy, a, b, tv);
              smp = sample_quadf(C, w, h, fadd(sx, u), syv);
            }
            const float residual = fsub(smp, tv);
            b1 = dadd(b1, (double)fmul(a, residual));
            b2 = dadd(b2, (double)fmul(b, residual));
          }
        }
        float du = __double2float_rn(dmul(-dsub(dmul(gyy, b1), dmul(gxy, b2)), inv_det));
        float dv = __double2float_rn(dmul(-dsub(dmul(gxx, b2), dmul(gxy, b1)), inv_det));
        du = clamp_ref(du, -max_step, max_step);
        dv = clamp_ref(dv, -max_step, max_step);
        u = fadd(u, du);
        v = fadd(v, dv);
        if (fabsf(u) > diverge_limit || fabsf(v) > diverge_limit) {
          lost = true;
          break;
        }
        if (fadd(fmul(du, du), fmul(dv, dv)) < 1e-6f) break;
      }
    }
    const float fx = fadd((float)ptx, u);
    const float fy = fadd((float)pty, v);
    if (!solved_any || fx < 0.0f || fx > fsub(w0, 1.0f) || fy < 0.0f || fy > fsub(h0, 1.0f)) lost = true;
    disp[pi] = make_float2(u, v);
    status[pi] = lost ? 0 : 1;
  }
}

// ---------------------------------------------------------------- launches

void launch_pyramid(const PyramidParams& p, int n_frames, cudaStream_t s) {
  if (n_frames <= 0) return;
  for (int l = 0; l < p.levels; ++l) {
    const int w = p.dims[l].w;
    if (l == 0 && p.u8_level0 && p.quad_u8.base && !p.tex[0].base && (w & 3) == 0 &&
        ((uintptr_t)p.frames.base & 3) == 0 && ((uintptr_t)p.quad_u8.base & 15) == 0 &&
        ((uintptr_t)p.tex8.base & 15) == 0) {
      dim3 g((w / 4 + 127) / 128, (p.dims[0].h + kPyrRows - 1) / kPyrRows, n_frames);
      if (p.tex8.base) quad_level0_kernel<true><<<g, 128, 0, s>>>(p);
      else quad_level0_kernel<false><<<g, 128, 0, s>>>(p);
      continue;
    }
    dim3 g((w + 127) / 128, (p.dims[l].h + kPyrRows - 1) / kPyrRows, n_frames);
    pyramid_level_kernel<<<g, 128, 0, s>>>(p, l);
  }
}

void launch_build_quad(const uint8_t* src, uint32_t* dst, int w, int h, cudaStream_t s) {
  dim3 g((w + 127) / 128, h);
  build_quad_kernel<<<g, 128, 0, s>>>(src, dst, w, h);
}

void launch_dense_lk(const DenseLKParams& p, int n_pairs, cudaStream_t s) {
  if (n_pairs <= 0) return;
  // patch rows [jt0, jt1): jt0 a multiple of the tile height
  dim3 grid((p.g.ncx + kLKTileX - 1) / kLKTileX, (p.jt1 - p.jt0 + kLKTileY - 1) / kLKTileY, n_pairs);
  const int r = p.radius;
  const size_t sm = dense_lk_smem(r);
  for (const void* f : {(const void*)dense_lk_warp_kernel<4, false>, (const void*)dense_lk_warp_kernel<6, false>,
                        (const void*)dense_lk_warp_kernel<4, true>, (const void*)dense_lk_warp_kernel<6, true>,
                        (const void*)dense_lk_tile_kernel<0>, (const void*)dense_lk_tile_kernel<4>,
                        (const void*)dense_lk_tile_kernel<6>})
    set_max_dynamic_smem(f, 200 * 1024);
  const bool inside = p.g.w > 2 * r + 1 && p.g.h > 2 * r + 1;  // no template clamping
  if (p.u8 && !((r == 4 || r == 6) && inside)) return;  // host guarantees the warp form for u8 levels
  if (r == 4 && inside && p.u8)
    dense_lk_warp_kernel<4, true><<<grid, kLKThreads, LKWarp<4>::floats * sizeof(float), s>>>(p);
  else if (r == 6 && inside && p.u8)
    dense_lk_warp_kernel<6, true><<<grid, kLKThreads, LKWarp<6>::floats * sizeof(float), s>>>(p);
  else if (r == 4 && inside)
    dense_lk_warp_kernel<4, false><<<grid, kLKThreads, LKWarp<4>::floats * sizeof(float), s>>>(p);
  else if (r == 6 && inside)
    dense_lk_warp_kernel<6, false><<<grid, kLKThreads, LKWarp<6>::floats * sizeof(float), s>>>(p);
  else if (r == 4) dense_lk_tile_kernel<4><<<grid, kLKThreads, sm, s>>>(p);
  else if (r == 6) dense_lk_tile_kernel<6><<<grid, kLKThreads, sm, s>>>(p);
  else if (sm <= 200 * 1024) dense_lk_tile_kernel<0><<<grid, kLKThreads, sm, s>>>(p);
  else dense_lk_global_kernel<<<dim3((p.g.ncx * (p.jt1 - p.jt0) + 127) / 128, n_pairs), 128, 0, s>>>(p);
}

void launch_densify(const GridGeom& g, float* du, float* dv, cudaStream_t s) {
  dim3 grid((g.w + 127) / 128, g.h);
  densify_kernel<<<grid, 128, 0, s>>>(g, du, dv);
}

void launch_sparse_lk(const SparseLKParams& p, int max_points, int n_pairs, cudaStream_t s) {
  if (n_pairs <= 0) return;
  int blocks = (max_points + 127) / 128;
  const int cap = (148 * 16 + n_pairs - 1) / n_pairs;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  sparse_lk_kernel<<<dim3(blocks, n_pairs), 128, 0, s>>>(p);
}

}  // namespace evsim_gpu
