// flow_kernels.cu — image pyramid, dense patch-grid Lucas–Kanade, sparse
// pyramidal Lucas–Kanade (sm_100a).
//
// Replaces src/flow.cpp of the reference (/root/reference/proj).  Every
// float/double operation keeps the reference's operation order and rounding
// (see evsim_device.cuh); fp64 sums are accumulated in the reference's k-order
// by one thread per patch / point, so results are bit-identical.
#include "evsim_device.cuh"
#include "kernels.h"

namespace evsim_gpu {

// ---------------------------------------------------------------- pyramid

// to_float  flow.cpp:23-27
__global__ void to_float_kernel(const uint8_t* __restrict__ src, float* __restrict__ dst, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = (float)src[i];
}

// downsample  flow.cpp:30-42: 0.25f * (((a + b) + c) + d), odd edges replicate
__global__ void downsample_kernel(const float* __restrict__ src, LevelDims sd, float* __restrict__ dst,
                                  LevelDims dd) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= dd.w || y >= dd.h) return;
  const int x0 = 2 * x, y0 = 2 * y;
  const int x1 = min(2 * x + 1, sd.w - 1);
  const int y1 = min(2 * y + 1, sd.h - 1);
  const float* r0 = src + (size_t)y0 * sd.w;
  const float* r1 = src + (size_t)y1 * sd.w;
  const float s = fadd(fadd(fadd(r0[x0], r0[x1]), r1[x0]), r1[x1]);
  dst[(size_t)y * dd.w + x] = fmul(0.25f, s);
}

// Quad image: the four bilinear taps of sample_u8 (simulate.cpp:10-26) per pixel.
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
// sample of the densified coarse field, divided by the level ratio.
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

// solve_level's per-patch loop (flow.cpp:170-215), one thread per patch.
// The fp64 sums run in the reference's (oy, ox) order.
__global__ void __launch_bounds__(128) dense_lk_kernel(DenseLKParams p) {
  const int pid = blockIdx.x * blockDim.x + threadIdx.x;
  const GridGeom& g = p.g;
  if (pid >= g.ncx * g.ncy) return;
  const int i = pid % g.ncx;
  const int j = pid / g.ncx;
  const int cx = __ldg(g.cx + i);
  const int cy = __ldg(g.cy + j);
  const int w = g.w, h = g.h, r = p.radius;
  float u = 0.0f, v = 0.0f;
  if (p.has_coarse) upsample_at(p.coarse, w, h, cx, cy, u, v);

  double gxx = 0.0, gxy = 0.0, gyy = 0.0;
  for (int oy = -r; oy <= r; ++oy) {
    const int py = clampi(cy + oy, 0, h - 1);
    for (int ox = -r; ox <= r; ++ox) {
      const int px = clampi(cx + ox, 0, w - 1);
      const float a = grad_x(p.prev, w, px, py);
      const float b = grad_y(p.prev, w, h, px, py);
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
          const float a = grad_x(p.prev, w, px, py);
          const float b = grad_y(p.prev, w, h, px, py);
          const float tval = __ldg(p.prev + (size_t)py * w + px);
          const float residual = fsub(sample_f32(p.curr, w, h, fadd((float)px, u), syv), tval);
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
  g.pu[pid] = u;
  g.pv[pid] = v;
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

// sample() of the materialised gradient images (flow.cpp:328-334): gradients
// evaluated at the four taps on the fly.
__device__ __forceinline__ void sample_grads(const float* __restrict__ im, int w, int h, float sx, float sy,
                                             float& a, float& b, float& val) {
  const Tap t = make_tap(sx, sy, w, h);
  const float gx00 = grad_x(im, w, t.x0, t.y0), gx10 = grad_x(im, w, t.x1, t.y0);
  const float gx01 = grad_x(im, w, t.x0, t.y1), gx11 = grad_x(im, w, t.x1, t.y1);
  const float gy00 = grad_y(im, w, h, t.x0, t.y0), gy10 = grad_y(im, w, h, t.x1, t.y0);
  const float gy01 = grad_y(im, w, h, t.x0, t.y1), gy11 = grad_y(im, w, h, t.x1, t.y1);
  const float* r0 = im + (size_t)t.y0 * w;
  const float* r1 = im + (size_t)t.y1 * w;
  a = lerp_ref(lerp_ref(gx00, gx10, t.fx), lerp_ref(gx01, gx11, t.fx), t.fy);
  b = lerp_ref(lerp_ref(gy00, gy10, t.fx), lerp_ref(gy01, gy11, t.fx), t.fy);
  val = lerp_ref(lerp_ref(__ldg(r0 + t.x0), __ldg(r0 + t.x1), t.fx),
                 lerp_ref(__ldg(r1 + t.x0), __ldg(r1 + t.x1), t.fx), t.fy);
}

// estimate_sparse_flow's per-point loop (flow.cpp:309-380), one thread per point.
__global__ void __launch_bounds__(128) sparse_lk_kernel(SparseLKParams p) {
  const int64_t M = p.n_points ? (int64_t)*p.n_points : p.n_points_host;
  const int r = p.radius;
  const int patch_pixels = (2 * r + 1) * (2 * r + 1);
  const float max_step = (float)r;
  const float diverge_limit = fmul(2.0f, (float)max(p.w0, p.h0));
  const float w0 = (float)p.w0, h0 = (float)p.h0;
  for (int64_t pi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pi < M;
       pi += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t idx = p.points[pi];
    const int ptx = (int)(idx % (uint32_t)p.w0);
    const int pty = (int)(idx / (uint32_t)p.w0);
    float u = 0.0f, v = 0.0f;
    bool lost = false, solved_any = false;
    for (int l = p.levels - 1; l >= 0 && !lost; --l) {
      const int w = p.dims[l].w, h = p.dims[l].h;
      const float* P = p.prev[l];
      const float* C = p.curr[l];
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
          sample_grads(P, w, h, fadd(px, (float)ox), sy, a, b, tv);
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
            sample_grads(P, w, h, sx, sy, a, b, tv);
            const float residual = fsub(sample_f32(C, w, h, fadd(sx, u), syv), tv);
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
    p.disp[pi] = make_float2(u, v);
    p.status[pi] = lost ? 0 : 1;
  }
}

// ---------------------------------------------------------------- launches

void launch_to_float(const uint8_t* src, float* dst, int64_t n, cudaStream_t s) {
  to_float_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(src, dst, n);
}

void launch_downsample(const float* src, LevelDims sd, float* dst, LevelDims dd, cudaStream_t s) {
  dim3 b(32, 8), g((dd.w + 31) / 32, (dd.h + 7) / 8);
  downsample_kernel<<<g, b, 0, s>>>(src, sd, dst, dd);
}

void launch_build_quad(const uint8_t* src, uint32_t* dst, int w, int h, cudaStream_t s) {
  dim3 g((w + 127) / 128, h);
  build_quad_kernel<<<g, 128, 0, s>>>(src, dst, w, h);
}

void launch_dense_lk(const DenseLKParams& p, cudaStream_t s) {
  const int n = p.g.ncx * p.g.ncy;
  dense_lk_kernel<<<(n + 127) / 128, 128, 0, s>>>(p);
}

void launch_densify(const GridGeom& g, float* du, float* dv, cudaStream_t s) {
  dim3 grid((g.w + 127) / 128, g.h);
  densify_kernel<<<grid, 128, 0, s>>>(g, du, dv);
}

void launch_sparse_lk(const SparseLKParams& p, int max_points, cudaStream_t s) {
  int blocks = (max_points + 127) / 128;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  sparse_lk_kernel<<<blocks, 128, 0, s>>>(p);
}

}  // namespace evsim_gpu
