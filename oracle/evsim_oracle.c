/*
 * evsim_oracle.c — TEST INFRASTRUCTURE ONLY (see evsim_oracle.h).
 *
 * Plain-C restatement of the reference hot path.  Every function names the
 * reference file:line it restates (paths relative to /root/reference/proj).
 * The operation order of every float/double expression is kept exactly as in
 * the reference so the results are bit-identical on x86-64 without FMA.
 */
#include "evsim_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* errors                                                                    */

static _Thread_local char g_err[512];

const char* evsim_oracle_last_error(void) { return g_err; }

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

/* ------------------------------------------------------------------------ */
/* small helpers                                                             */

static int imin(int a, int b) { return a < b ? a : b; }
static int imax(int a, int b) { return a > b ? a : b; }
/* std::clamp semantics (lo if v < lo, hi if hi < v, else v; NaN passes). */
static float clampf_ref(float v, float lo, float hi) { return (v < lo) ? lo : ((hi < v) ? hi : v); }
static int clampi(int v, int lo, int hi) { return (v < lo) ? lo : ((hi < v) ? hi : v); }

/* sub_interval_end  include/evsim/simulate.hpp:15-19 */
static int64_t sub_interval_end(int64_t t0, int64_t t1, int k, int n_steps) {
  const int64_t dt = t1 - t0;
  const int64_t num = (int64_t)k * dt;
  return t0 + (num + n_steps - 1) / n_steps;
}

void evsim_oracle_log_lut(float* lut) {
  for (int i = 0; i < 256; ++i) lut[i] = logf((float)i / 255.0f + 1e-3f);
}

/* ------------------------------------------------------------------------ */
/* event vector + ordering                                                   */

typedef struct {
  evsim_event* v;
  int64_t n, cap;
} evvec;

static void ev_push(evvec* e, uint16_t x, uint16_t y, int64_t t, int8_t p) {
  if (e->n == e->cap) {
    e->cap = e->cap ? e->cap * 2 : 1024;
    e->v = (evsim_event*)realloc(e->v, (size_t)e->cap * sizeof(evsim_event));
  }
  evsim_event* d = &e->v[e->n++];
  memset(d, 0, sizeof *d);
  d->x = x;
  d->y = y;
  d->t = t;
  d->p = p;
}

/* event_order  include/evsim/types.hpp:64-69 */
static int event_less(const evsim_event* a, const evsim_event* b) {
  if (a->t != b->t) return a->t < b->t;
  if (a->y != b->y) return a->y < b->y;
  if (a->x != b->x) return a->x < b->x;
  return a->p < b->p;
}

static void merge_sort(evsim_event* a, evsim_event* tmp, int64_t n) {
  if (n < 2) return;
  const int64_t m = n / 2;
  merge_sort(a, tmp, m);
  merge_sort(a + m, tmp, n - m);
  int64_t i = 0, j = m, k = 0;
  while (i < m && j < n) {
    if (event_less(&a[j], &a[i])) tmp[k++] = a[j++]; /* stable: left wins ties */
    else tmp[k++] = a[i++];
  }
  while (i < m) tmp[k++] = a[i++];
  while (j < n) tmp[k++] = a[j++];
  memcpy(a, tmp, (size_t)n * sizeof *a);
}

/* finalize  src/simulate.cpp:36-40: stable sort only when unsorted */
static void finalize(evvec* e) {
  int sorted = 1;
  for (int64_t i = 1; i < e->n; ++i) {
    if (event_less(&e->v[i], &e->v[i - 1])) { sorted = 0; break; }
  }
  if (sorted) return;
  evsim_event* tmp = (evsim_event*)malloc((size_t)e->n * sizeof *tmp);
  merge_sort(e->v, tmp, e->n);
  free(tmp);
}

/* ------------------------------------------------------------------------ */
/* optical flow  src/flow.cpp                                                */

typedef struct {
  int w, h;
  float* v;
} img;

static img img_new(int w, int h) {
  img im = {w, h, (float*)calloc((size_t)w * h, sizeof(float))};
  return im;
}
static void img_free(img* im) { free(im->v); im->v = NULL; }
#define AT(im, x, y) ((im).v[(size_t)(y) * (im).w + (x)])

/* to_float  flow.cpp:23-27 */
static img to_float(const uint8_t* px, int w, int h) {
  img im = img_new(w, h);
  for (size_t i = 0; i < (size_t)w * h; ++i) im.v[i] = (float)px[i];
  return im;
}

/* downsample  flow.cpp:30-42 */
static img downsample(const img* src) {
  img dst = img_new((src->w + 1) / 2, (src->h + 1) / 2);
  for (int y = 0; y < dst.h; ++y) {
    const int y0 = 2 * y;
    const int y1 = imin(2 * y + 1, src->h - 1);
    for (int x = 0; x < dst.w; ++x) {
      const int x0 = 2 * x;
      const int x1 = imin(2 * x + 1, src->w - 1);
      AT(dst, x, y) = 0.25f * (AT(*src, x0, y0) + AT(*src, x1, y0) + AT(*src, x0, y1) + AT(*src, x1, y1));
    }
  }
  return dst;
}

/* sample  flow.cpp:45-57 */
static float sample(const img* im, float x, float y) {
  x = clampf_ref(x, 0.0f, (float)(im->w - 1));
  y = clampf_ref(y, 0.0f, (float)(im->h - 1));
  const int x0 = (int)x;
  const int y0 = (int)y;
  const int x1 = imin(x0 + 1, im->w - 1);
  const int y1 = imin(y0 + 1, im->h - 1);
  const float fx = x - (float)x0;
  const float fy = y - (float)y0;
  const float top = AT(*im, x0, y0) + fx * (AT(*im, x1, y0) - AT(*im, x0, y0));
  const float bot = AT(*im, x0, y1) + fx * (AT(*im, x1, y1) - AT(*im, x0, y1));
  return top + fy * (bot - top);
}

/* gradients  flow.cpp:60-73 */
static void gradients(const img* im, img* gx, img* gy) {
  *gx = img_new(im->w, im->h);
  *gy = img_new(im->w, im->h);
  for (int y = 0; y < im->h; ++y) {
    const int ym = imax(y - 1, 0);
    const int yp = imin(y + 1, im->h - 1);
    for (int x = 0; x < im->w; ++x) {
      const int xm = imax(x - 1, 0);
      const int xp = imin(x + 1, im->w - 1);
      AT(*gx, x, y) = 0.5f * (AT(*im, xp, y) - AT(*im, xm, y));
      AT(*gy, x, y) = 0.5f * (AT(*im, x, yp) - AT(*im, x, ym));
    }
  }
}

/* effective_levels  flow.cpp:75-79 (kMinPyramidExtent = 8, flow.cpp:10) */
static int effective_levels(int requested, int w, int h) {
  int levels = imax(1, requested);
  while (levels > 1 && (imin(w, h) >> (levels - 1)) < 8) --levels;
  return levels;
}

/* build_pyramid  flow.cpp:81-87 */
static img* build_pyramid(const uint8_t* px, int w, int h, int levels) {
  img* pyr = (img*)calloc((size_t)levels, sizeof(img));
  pyr[0] = to_float(px, w, h);
  for (int l = 1; l < levels; ++l) pyr[l] = downsample(&pyr[l - 1]);
  return pyr;
}
static void free_pyramid(img* pyr, int levels) {
  for (int l = 0; l < levels; ++l) img_free(&pyr[l]);
  free(pyr);
}

/* min_eigenvalue  flow.cpp:89-93 */
static double min_eigenvalue(double gxx, double gxy, double gyy) {
  const double trace = gxx + gyy;
  const double dd = (gxx - gyy) * (gxx - gyy) + 4.0 * gxy * gxy;
  const double disc = sqrt(dd > 0.0 ? dd : 0.0); /* std::max(0.0, dd) */
  return 0.5 * (trace - disc);
}

/* patch_centers  flow.cpp:97-107; returns count, centers malloc'd */
static int patch_centers(int extent, int radius, int stride, int** out) {
  int cap = extent / (stride > 0 ? stride : 1) + 3;
  int* c = (int*)malloc((size_t)cap * sizeof(int));
  int n = 0;
  if (extent <= 2 * radius + 1) {
    c[n++] = (extent - 1) / 2;
    *out = c;
    return n;
  }
  const int last = extent - 1 - radius;
  for (int v = radius; v <= last; v += stride) c[n++] = v;
  if (c[n - 1] != last) c[n++] = last;
  *out = c;
  return n;
}

/* interp_table  flow.cpp:111-128 */
static void interp_table(const int* centers, int nc, int extent, int* idx, float* wgt) {
  for (int x = 0; x < extent; ++x) { idx[x] = 0; wgt[x] = 0.0f; }
  if (nc < 2) return;
  int j = 0;
  for (int x = 0; x < extent; ++x) {
    if (x <= centers[0]) continue;
    if (x >= centers[nc - 1]) {
      idx[x] = nc - 2;
      wgt[x] = 1.0f;
      continue;
    }
    while (j + 2 < nc && centers[j + 1] <= x) ++j;
    idx[x] = j;
    wgt[x] = (float)(x - centers[j]) / (float)(centers[j + 1] - centers[j]);
  }
}

typedef struct {
  int w, h;
  float* du;
  float* dv;
} flowf;

static flowf flow_new(int w, int h) {
  flowf f = {w, h, (float*)calloc((size_t)w * h, sizeof(float)),
             (float*)calloc((size_t)w * h, sizeof(float))};
  return f;
}
static void flow_free(flowf* f) { free(f->du); free(f->dv); f->du = f->dv = NULL; }

/* upsample_flow  flow.cpp:130-147 */
static flowf upsample_flow(const flowf* coarse, int w, int h) {
  flowf fine = flow_new(w, h);
  const img cu = {coarse->w, coarse->h, coarse->du};
  const img cv = {coarse->w, coarse->h, coarse->dv};
  const float rx = (float)coarse->w / (float)w;
  const float ry = (float)coarse->h / (float)h;
  size_t i = 0;
  for (int y = 0; y < h; ++y) {
    const float sy = ((float)y + 0.5f) * ry - 0.5f;
    for (int x = 0; x < w; ++x, ++i) {
      const float sx = ((float)x + 0.5f) * rx - 0.5f;
      fine.du[i] = sample(&cu, sx, sy) / rx;
      fine.dv[i] = sample(&cv, sx, sy) / ry;
    }
  }
  return fine;
}

/* solve_level  flow.cpp:152-247 (kMinEigPerPixel = 1e-4, flow.cpp:9) */
static flowf solve_level(const img* prev, const img* gx, const img* gy, const img* curr,
                         const flowf* init, int iterations, int r) {
  const int w = prev->w;
  const int h = prev->h;
  const int stride = imax(1, r);
  int *cxs, *cys;
  const int ncx = patch_centers(w, r, stride, &cxs);
  const int ncy = patch_centers(h, r, stride, &cys);
  const int patch_pixels = (2 * r + 1) * (2 * r + 1);
  const float max_step = (float)r;

  float* pu = (float*)malloc((size_t)ncx * ncy * sizeof(float));
  float* pv = (float*)malloc((size_t)ncx * ncy * sizeof(float));
  float* tgx = (float*)malloc((size_t)patch_pixels * sizeof(float));
  float* tgy = (float*)malloc((size_t)patch_pixels * sizeof(float));
  float* tval = (float*)malloc((size_t)patch_pixels * sizeof(float));
  int* txs = (int*)malloc((size_t)patch_pixels * sizeof(int));
  int* tys = (int*)malloc((size_t)patch_pixels * sizeof(int));

  for (int j = 0; j < ncy; ++j) {
    const int cy = cys[j];
    for (int i = 0; i < ncx; ++i) {
      const int cx = cxs[i];
      float u = init->du[(size_t)cy * init->w + cx];
      float v = init->dv[(size_t)cy * init->w + cx];
      double gxx = 0.0, gxy = 0.0, gyy = 0.0;
      int n = 0;
      for (int oy = -r; oy <= r; ++oy) {
        const int py = clampi(cy + oy, 0, h - 1);
        for (int ox = -r; ox <= r; ++ox, ++n) {
          const int px = clampi(cx + ox, 0, w - 1);
          const float a = AT(*gx, px, py);
          const float b = AT(*gy, px, py);
          tgx[n] = a;
          tgy[n] = b;
          tval[n] = AT(*prev, px, py);
          txs[n] = px;
          tys[n] = py;
          gxx += a * a;
          gxy += a * b;
          gyy += b * b;
        }
      }
      if (min_eigenvalue(gxx, gxy, gyy) > 1e-4 * patch_pixels) {
        const double inv_det = 1.0 / (gxx * gyy - gxy * gxy);
        for (int it = 0; it < iterations; ++it) {
          double b1 = 0.0, b2 = 0.0;
          for (int k = 0; k < patch_pixels; ++k) {
            const float residual = sample(curr, (float)txs[k] + u, (float)tys[k] + v) - tval[k];
            b1 += tgx[k] * residual;
            b2 += tgy[k] * residual;
          }
          float du = (float)(-(gyy * b1 - gxy * b2) * inv_det);
          float dv = (float)(-(gxx * b2 - gxy * b1) * inv_det);
          du = clampf_ref(du, -max_step, max_step);
          dv = clampf_ref(dv, -max_step, max_step);
          u += du;
          v += dv;
        }
      }
      pu[(size_t)j * ncx + i] = u;
      pv[(size_t)j * ncx + i] = v;
    }
  }

  int* ix = (int*)malloc((size_t)w * sizeof(int));
  int* iy = (int*)malloc((size_t)h * sizeof(int));
  float* wx = (float*)malloc((size_t)w * sizeof(float));
  float* wy = (float*)malloc((size_t)h * sizeof(float));
  interp_table(cxs, ncx, w, ix, wx);
  interp_table(cys, ncy, h, iy, wy);
#define GRID(g, i_, j_) (g)[(size_t)imin((j_), ncy - 1) * ncx + imin((i_), ncx - 1)]
  flowf out = flow_new(w, h);
  size_t idx = 0;
  for (int y = 0; y < h; ++y) {
    const int j = iy[y];
    const float fy = wy[y];
    for (int x = 0; x < w; ++x, ++idx) {
      const int i = ix[x];
      const float fx = wx[x];
      const float u_top = GRID(pu, i, j) + fx * (GRID(pu, i + 1, j) - GRID(pu, i, j));
      const float u_bot = GRID(pu, i, j + 1) + fx * (GRID(pu, i + 1, j + 1) - GRID(pu, i, j + 1));
      const float v_top = GRID(pv, i, j) + fx * (GRID(pv, i + 1, j) - GRID(pv, i, j));
      const float v_bot = GRID(pv, i, j + 1) + fx * (GRID(pv, i + 1, j + 1) - GRID(pv, i, j + 1));
      out.du[idx] = u_top + fy * (u_bot - u_top);
      out.dv[idx] = v_top + fy * (v_bot - v_top);
    }
  }
#undef GRID
  free(ix); free(iy); free(wx); free(wy);
  free(pu); free(pv); free(tgx); free(tgy); free(tval); free(txs); free(tys);
  free(cxs); free(cys);
  return out;
}

static int check_preset(int levels, int iters, int radius) {
  /* FlowPreset::validate  include/evsim/flow.hpp:50-54 */
  if (levels < 1 || iters < 1 || radius < 1)
    return fail(EVSIM_GPU_INVALID_ARGUMENT, "FlowPreset: all fields must be >= 1");
  return 0;
}

/* estimate_dense_flow  flow.cpp:260-276 */
int evsim_oracle_dense_flow(const uint8_t* prev, const uint8_t* curr, int32_t w, int32_t h,
                            int32_t levels_req, int32_t iters, int32_t radius, float* du,
                            float* dv) {
  int rc = check_preset(levels_req, iters, radius);
  if (rc) return rc;
  if (w <= 0 || h <= 0 || !prev || !curr)
    return fail(EVSIM_GPU_INVALID_ARGUMENT, "estimate_dense_flow: empty frame");
  const int levels = effective_levels(levels_req, w, h);
  img* pp = build_pyramid(prev, w, h, levels);
  img* pc = build_pyramid(curr, w, h, levels);
  flowf flow = flow_new(pp[levels - 1].w, pp[levels - 1].h);
  for (int l = levels - 1; l >= 0; --l) {
    if (l != levels - 1) {
      flowf up = upsample_flow(&flow, pp[l].w, pp[l].h);
      flow_free(&flow);
      flow = up;
    }
    img gx, gy;
    gradients(&pp[l], &gx, &gy);
    flowf next = solve_level(&pp[l], &gx, &gy, &pc[l], &flow, iters, radius);
    flow_free(&flow);
    flow = next;
    img_free(&gx);
    img_free(&gy);
  }
  memcpy(du, flow.du, (size_t)w * h * sizeof(float));
  memcpy(dv, flow.dv, (size_t)w * h * sizeof(float));
  flow_free(&flow);
  free_pyramid(pp, levels);
  free_pyramid(pc, levels);
  return 0;
}

/* estimate_sparse_flow  flow.cpp:278-381 */
int evsim_oracle_sparse_flow(const uint8_t* prev, const uint8_t* curr, int32_t w, int32_t h,
                             int32_t levels_req, int32_t iters, int32_t r, const int32_t* pts,
                             int64_t n_points, float* disp, uint8_t* status) {
  int rc = check_preset(levels_req, iters, r);
  if (rc) return rc;
  if (w <= 0 || h <= 0 || !prev || !curr)
    return fail(EVSIM_GPU_INVALID_ARGUMENT, "estimate_sparse_flow: empty frame");
  for (int64_t i = 0; i < n_points; ++i) {
    const int px = pts[2 * i], py = pts[2 * i + 1];
    if (px < 0 || px >= w || py < 0 || py >= h)
      return fail(EVSIM_GPU_INVALID_ARGUMENT, "estimate_sparse_flow: point outside frame bounds");
  }
  for (int64_t i = 0; i < n_points; ++i) {
    disp[2 * i] = 0.0f;
    disp[2 * i + 1] = 0.0f;
    status[i] = 0;
  }
  if (n_points == 0) return 0;

  const int levels = effective_levels(levels_req, w, h);
  img* pp = build_pyramid(prev, w, h, levels);
  img* pc = build_pyramid(curr, w, h, levels);
  img* pgx = (img*)calloc((size_t)levels, sizeof(img));
  img* pgy = (img*)calloc((size_t)levels, sizeof(img));
  for (int l = 0; l < levels; ++l) gradients(&pp[l], &pgx[l], &pgy[l]);

  const int patch_pixels = (2 * r + 1) * (2 * r + 1);
  const float max_step = (float)r;
  const float diverge_limit = 2.0f * (float)imax(w, h);
  float* tgx = (float*)malloc((size_t)patch_pixels * sizeof(float));
  float* tgy = (float*)malloc((size_t)patch_pixels * sizeof(float));
  float* tval = (float*)malloc((size_t)patch_pixels * sizeof(float));
  const float w0 = (float)w;
  const float h0 = (float)h;

  for (int64_t pi = 0; pi < n_points; ++pi) {
    float u = 0.0f, v = 0.0f;
    int lost = 0, solved_any = 0;
    const int ptx = pts[2 * pi], pty = pts[2 * pi + 1];
    for (int l = levels - 1; l >= 0 && !lost; --l) {
      const img* P = &pp[l];
      const img* C = &pc[l];
      const float px = ((float)ptx + 0.5f) * ((float)P->w / w0) - 0.5f;
      const float py = ((float)pty + 0.5f) * ((float)P->h / h0) - 0.5f;
      if (l != levels - 1) {
        u *= (float)P->w / (float)pp[l + 1].w;
        v *= (float)P->h / (float)pp[l + 1].h;
      }
      double gxx = 0.0, gxy = 0.0, gyy = 0.0;
      int n = 0;
      for (int oy = -r; oy <= r; ++oy) {
        for (int ox = -r; ox <= r; ++ox, ++n) {
          const float sx = px + (float)ox;
          const float sy = py + (float)oy;
          const float a = sample(&pgx[l], sx, sy);
          const float b = sample(&pgy[l], sx, sy);
          tgx[n] = a;
          tgy[n] = b;
          tval[n] = sample(P, sx, sy);
          gxx += a * a;
          gxy += a * b;
          gyy += b * b;
        }
      }
      if (min_eigenvalue(gxx, gxy, gyy) <= 1e-4 * patch_pixels) continue;
      solved_any = 1;
      const double inv_det = 1.0 / (gxx * gyy - gxy * gxy);
      for (int it = 0; it < iters; ++it) {
        double b1 = 0.0, b2 = 0.0;
        int k = 0;
        for (int oy = -r; oy <= r; ++oy) {
          for (int ox = -r; ox <= r; ++ox, ++k) {
            const float residual = sample(C, px + (float)ox + u, py + (float)oy + v) - tval[k];
            b1 += tgx[k] * residual;
            b2 += tgy[k] * residual;
          }
        }
        float du = (float)(-(gyy * b1 - gxy * b2) * inv_det);
        float dv = (float)(-(gxx * b2 - gxy * b1) * inv_det);
        du = clampf_ref(du, -max_step, max_step);
        dv = clampf_ref(dv, -max_step, max_step);
        u += du;
        v += dv;
        if (fabsf(u) > diverge_limit || fabsf(v) > diverge_limit) {
          lost = 1;
          break;
        }
        if (du * du + dv * dv < 1e-6f) break;
      }
    }
    const float fx = (float)ptx + u;
    const float fy = (float)pty + v;
    if (!solved_any || fx < 0.0f || fx > w0 - 1.0f || fy < 0.0f || fy > h0 - 1.0f) lost = 1;
    disp[2 * pi] = u;
    disp[2 * pi + 1] = v;
    status[pi] = lost ? 0 : 1;
  }
  free(tgx); free(tgy); free(tval);
  for (int l = 0; l < levels; ++l) { img_free(&pgx[l]); img_free(&pgy[l]); }
  free(pgx); free(pgy);
  free_pyramid(pp, levels);
  free_pyramid(pc, levels);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* interpolation + chain  src/simulate.cpp                                   */

/* sample_u8  simulate.cpp:10-26 */
static float sample_u8(const uint8_t* f, int w, int h, float x, float y) {
  x = clampf_ref(x, 0.0f, (float)(w - 1));
  y = clampf_ref(y, 0.0f, (float)(h - 1));
  const int x0 = (int)x;
  const int y0 = (int)y;
  const int x1 = imin(x0 + 1, w - 1);
  const int y1 = imin(y0 + 1, h - 1);
  const float fx = x - (float)x0;
  const float fy = y - (float)y0;
  const float a00 = f[(size_t)y0 * w + x0];
  const float a10 = f[(size_t)y0 * w + x1];
  const float a01 = f[(size_t)y1 * w + x0];
  const float a11 = f[(size_t)y1 * w + x1];
  const float top = a00 + fx * (a10 - a00);
  const float bot = a01 + fx * (a11 - a01);
  return top + fy * (bot - top);
}

/* interpolate_frames  simulate.cpp:91-121 */
int evsim_oracle_interpolate_frames(const uint8_t* prev, const uint8_t* curr, int32_t w, int32_t h,
                                    int64_t t_prev, int64_t t_curr, const float* du,
                                    const float* dv, int32_t n, uint8_t* out, int64_t* out_t) {
  if (n < 0) return fail(EVSIM_GPU_INVALID_ARGUMENT, "interpolate_frames: n must be >= 0");
  const size_t P = (size_t)w * h;
  for (int k = 1; k <= n; ++k) {
    const double alpha = (double)k / (double)(n + 1);
    const float fwd = (float)alpha;
    const float bwd = (float)(1.0 - alpha);
    uint8_t* f = out + (size_t)(k - 1) * P;
    out_t[k - 1] = sub_interval_end(t_prev, t_curr, k, n + 1);
    size_t i = 0;
    for (int y = 0; y < h; ++y) {
      for (int x = 0; x < w; ++x, ++i) {
        const float u = du[i];
        const float v = dv[i];
        const float from_prev = sample_u8(prev, w, h, (float)x - fwd * u, (float)y - fwd * v);
        const float from_curr = sample_u8(curr, w, h, (float)x + bwd * u, (float)y + bwd * v);
        f[i] = (uint8_t)lround((1.0 - alpha) * from_prev + alpha * from_curr);
      }
    }
  }
  return 0;
}

typedef struct {
  const evsim_gpu_config* cfg;
  const float* lut; /* log mode */
  float* ref;       /* log mode: per-pixel reference state, updated in place */
} chain_ctx;

/* threshold_events_into  src/core.cpp:21-46 applied to curr - prev
 * (difference_frame, src/core.cpp:5-19), or the log-mode rule. */
static void link_events(const chain_ctx* cx, const uint8_t* before, const uint8_t* after, int w,
                        int h, int64_t t, evvec* out) {
  const evsim_gpu_config* c = cx->cfg;
  const int magnitude = c->events_per_crossing == EVSIM_EVENTS_MAGNITUDE;
  if (c->contrast_mode == EVSIM_CONTRAST_LOG) {
    const float cp = c->c_pos_log, cn = c->c_neg_log;
    for (int y = 0; y < h; ++y) {
      for (int x = 0; x < w; ++x) {
        const size_t i = (size_t)y * w + x;
        const float lk = cx->lut[after[i]];
        const float d = lk - cx->ref[i];
        if (d > cp) {
          const int count = magnitude ? (int)floorf(d / cp) : 1;
          for (int k = 0; k < count; ++k) ev_push(out, (uint16_t)x, (uint16_t)y, t, 1);
          cx->ref[i] = lk;
        } else if (d < cn) {
          const int count = magnitude ? (int)floorf(d / cn) : 1;
          for (int k = 0; k < count; ++k) ev_push(out, (uint16_t)x, (uint16_t)y, t, -1);
          cx->ref[i] = lk;
        }
      }
    }
    return;
  }
  const int c_pos = c->c_pos, c_neg = c->c_neg;
  for (int y = 0; y < h; ++y) {
    for (int x = 0; x < w; ++x) {
      const size_t i = (size_t)y * w + x;
      const int v = (int)(int16_t)((int)after[i] - (int)before[i]);
      if (v > c_pos) {
        const int count = magnitude ? v / c_pos : 1;
        for (int k = 0; k < count; ++k) ev_push(out, (uint16_t)x, (uint16_t)y, t, 1);
      } else if (v < c_neg) {
        const int count = magnitude ? v / c_neg : 1;
        for (int k = 0; k < count; ++k) ev_push(out, (uint16_t)x, (uint16_t)y, t, -1);
      }
    }
  }
}

/* chain_pipeline + chain_events + finalize  simulate.cpp:44-69, 36-40 */
static void chain_pipeline(const chain_ctx* cx, const uint8_t* prev, int64_t t_prev,
                           const uint8_t* curr, int64_t t_curr, const uint8_t* inter,
                           const int64_t* inter_t, int n_inter, int w, int h, evvec* out) {
  const size_t P = (size_t)w * h;
  const int m = n_inter + (cx->cfg->include_endpoints ? 2 : 0);
  const uint8_t** frames = (const uint8_t**)malloc((size_t)(m > 0 ? m : 1) * sizeof(*frames));
  int64_t* ts = (int64_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(int64_t));
  int c = 0;
  if (cx->cfg->include_endpoints) { frames[c] = prev; ts[c++] = t_prev; }
  for (int k = 0; k < n_inter; ++k) { frames[c] = inter + (size_t)k * P; ts[c++] = inter_t[k]; }
  if (cx->cfg->include_endpoints) { frames[c] = curr; ts[c++] = t_curr; }
  for (int i = 1; i < m; ++i) link_events(cx, frames[i - 1], frames[i], w, h, ts[i], out);
  finalize(out);
  free(frames);
  free(ts);
}

/* dense_events_with_flow  simulate.cpp:123-128 */
static void dense_with_flow(const chain_ctx* cx, const uint8_t* prev, const uint8_t* curr, int w,
                            int h, int64_t t_prev, int64_t t_curr, const float* du,
                            const float* dv, evvec* out) {
  const int n = cx->cfg->n_interp;
  uint8_t* inter = (uint8_t*)malloc((size_t)(n > 0 ? n : 1) * w * h);
  int64_t* inter_t = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
  evsim_oracle_interpolate_frames(prev, curr, w, h, t_prev, t_curr, du, dv, n, inter, inter_t);
  chain_pipeline(cx, prev, t_prev, curr, t_curr, inter, inter_t, n, w, h, out);
  free(inter);
  free(inter_t);
}

/* sparse splat  simulate.cpp:163-201 */
static void sparse_with_flow(const chain_ctx* cx, const uint8_t* prev, const uint8_t* curr, int w,
                             int h, int64_t t_prev, int64_t t_curr, const int32_t* pts,
                             int64_t M, const float* disp, const uint8_t* status, evvec* out) {
  const int N = cx->cfg->n_interp;
  const size_t P = (size_t)w * h;
  uint8_t* inter = (uint8_t*)malloc((size_t)N * P);
  int64_t* inter_t = (int64_t*)malloc((size_t)N * sizeof(int64_t));
  int* claim_mark = (int*)malloc(P * sizeof(int));
  int* claim_change = (int*)calloc(P, sizeof(int));
  for (size_t i = 0; i < P; ++i) claim_mark[i] = -1;
  for (int k = 1; k <= N; ++k) {
    const float alpha = (float)k / (float)(N + 1);
    uint8_t* f = inter + (size_t)(k - 1) * P;
    memcpy(f, prev, P);
    inter_t[k - 1] = sub_interval_end(t_prev, t_curr, k, N + 1);
    for (int64_t j = 0; j < M; ++j) {
      if (!status[j]) continue;
      const int px = pts[2 * j], py = pts[2 * j + 1];
      const int tx = (int)lroundf((float)px + alpha * disp[2 * j]);
      const int ty = (int)lroundf((float)py + alpha * disp[2 * j + 1]);
      if (tx < 0 || tx >= w || ty < 0 || ty >= h) continue;
      const size_t idx = (size_t)ty * w + tx;
      const uint8_t value = prev[(size_t)py * w + px];
      const int change = abs((int)value - (int)prev[idx]);
      if (claim_mark[idx] != k) {
        claim_mark[idx] = k;
        claim_change[idx] = change;
        f[idx] = value;
      } else if (change > claim_change[idx]) {
        claim_change[idx] = change;
        f[idx] = value;
      }
    }
  }
  chain_pipeline(cx, prev, t_prev, curr, t_curr, inter, inter_t, N, w, h, out);
  free(inter); free(inter_t); free(claim_mark); free(claim_change);
}

/* difference_interp_events  simulate.cpp:212-285: d1 = the previous
 * interval's difference frame, d2 the newly completed one (t0, t1]. */
static int cmp_size(const void* a, const void* b) {
  const size_t x = *(const size_t*)a, y = *(const size_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

static void threshold_diff(const evsim_gpu_config* c, const int16_t* d, int w, int h, int64_t t, evvec* out) {
  /* threshold_events_into  core.cpp:21-46 */
  const int magnitude = c->events_per_crossing == EVSIM_EVENTS_MAGNITUDE;
  for (int y = 0; y < h; ++y) {
    for (int x = 0; x < w; ++x) {
      const int v = d[(size_t)y * w + x];
      if (v > c->c_pos) {
        const int count = magnitude ? v / c->c_pos : 1;
        for (int k = 0; k < count; ++k) ev_push(out, (uint16_t)x, (uint16_t)y, t, 1);
      } else if (v < c->c_neg) {
        const int count = magnitude ? v / c->c_neg : 1;
        for (int k = 0; k < count; ++k) ev_push(out, (uint16_t)x, (uint16_t)y, t, -1);
      }
    }
  }
}

static void diff_interp_events(const evsim_gpu_config* c, int levels, int iters, int radius,
                               const int16_t* d1, const int16_t* d2, int w, int h, int64_t t0,
                               int64_t t1, evvec* out) {
  const size_t P = (size_t)w * h;
  const int N = c->n_interp;
  const int magnitude = c->events_per_crossing == EVSIM_EVENTS_MAGNITUDE;
  /* active_points  simulate.cpp:78-87: scan order */
  int64_t M = 0;
  for (size_t i = 0; i < P; ++i) M += (d1[i] > c->c_pos || d1[i] < c->c_neg);
  if (M > 0 && N > 0) {
    int32_t* pts = (int32_t*)malloc((size_t)M * 2 * sizeof(int32_t));
    int16_t* val = (int16_t*)malloc((size_t)M * sizeof(int16_t));
    int64_t j = 0;
    for (int y = 0; y < h; ++y)
      for (int x = 0; x < w; ++x) {
        const int v = d1[(size_t)y * w + x];
        if (v > c->c_pos || v < c->c_neg) {
          pts[2 * j] = x;
          pts[2 * j + 1] = y;
          val[j++] = (int16_t)v;
        }
      }
    /* flow on magnitude images min(255, |d|) (simulate.cpp:223-233) */
    uint8_t* m1 = (uint8_t*)malloc(P);
    uint8_t* m2 = (uint8_t*)malloc(P);
    for (size_t i = 0; i < P; ++i) {
      m1[i] = (uint8_t)imin(255, abs((int)d1[i]));
      m2[i] = (uint8_t)imin(255, abs((int)d2[i]));
    }
    float* disp = (float*)malloc((size_t)M * 2 * sizeof(float));
    uint8_t* st = (uint8_t*)malloc((size_t)M);
    evsim_oracle_sparse_flow(m1, m2, w, h, levels, iters, radius, pts, M, disp, st);
    int* mark = (int*)malloc(P * sizeof(int));
    int16_t* inter = (int16_t*)malloc(P * sizeof(int16_t));
    size_t* touched = (size_t*)malloc((size_t)M * sizeof(size_t));
    for (size_t i = 0; i < P; ++i) mark[i] = -1;
    for (int k = 1; k <= N; ++k) {
      const float alpha = (float)k / (float)(N + 1);
      const int64_t t = sub_interval_end(t0, t1, k, N + 1);
      int64_t nt = 0;
      for (int64_t q = 0; q < M; ++q) {
        if (!st[q]) continue;
        const int tx = (int)lroundf((float)pts[2 * q] + alpha * disp[2 * q]);
        const int ty = (int)lroundf((float)pts[2 * q + 1] + alpha * disp[2 * q + 1]);
        if (tx < 0 || tx >= w || ty < 0 || ty >= h) continue;
        const size_t idx = (size_t)ty * w + tx;
        if (mark[idx] != k) {
          mark[idx] = k;
          inter[idx] = val[q];
          touched[nt++] = idx;
        } else if (abs((int)val[q]) > abs((int)inter[idx])) {
          inter[idx] = val[q];
        }
      }
      qsort(touched, (size_t)nt, sizeof(size_t), cmp_size);
      for (int64_t q = 0; q < nt; ++q) {
        const size_t idx = touched[q];
        const int v = inter[idx];
        const uint16_t ex = (uint16_t)(idx % (size_t)w), ey = (uint16_t)(idx / (size_t)w);
        if (v > c->c_pos) {
          int count = magnitude ? v / c->c_pos : 1;
          while (count-- > 0) ev_push(out, ex, ey, t, 1);
        } else if (v < c->c_neg) {
          int count = magnitude ? v / c->c_neg : 1;
          while (count-- > 0) ev_push(out, ex, ey, t, -1);
        }
      }
    }
    free(pts); free(val); free(m1); free(m2); free(disp); free(st); free(mark); free(inter); free(touched);
  }
  if (c->include_endpoints) threshold_diff(c, d2, w, h, t1, out); /* simulate.cpp:278-281 */
  finalize(out);
}

/* ------------------------------------------------------------------------ */
/* Simulator  include/evsim/simulate.hpp:60-94, src/simulate.cpp:306-347     */

struct evsim_oracle_sim {
  evsim_gpu_config cfg;
  int levels, iters, radius; /* resolved flow preset */
  int has_prev;
  int w, h;
  int64_t prev_t;
  uint8_t* prev;
  float* ref;
  int16_t* pdiff; /* difference_interp: the previous interval's difference frame */
  int has_pdiff;
  float lut[256];
  evvec ev;
};

static void resolve_preset(const evsim_gpu_config* c, int* levels, int* iters, int* radius) {
  if (c->pyramid_levels || c->iterations_per_level || c->patch_radius) {
    *levels = c->pyramid_levels;
    *iters = c->iterations_per_level;
    *radius = c->patch_radius;
  } else if (c->flow_preset == EVSIM_FLOW_HIGH_QUALITY) {
    *levels = 5; *iters = 16; *radius = 6; /* flow_preset(hq)  flow.hpp:57-59 */
  } else {
    *levels = 3; *iters = 2; *radius = 4;  /* flow_preset(lq) */
  }
}

static int validate_cfg(const evsim_gpu_config* c) {
  /* SimulatorConfig::validate  types.hpp:126-130 */
  if (c->c_pos <= 0) return fail(EVSIM_GPU_INVALID_ARGUMENT, "SimulatorConfig: c_pos must be > 0");
  if (c->c_neg >= 0) return fail(EVSIM_GPU_INVALID_ARGUMENT, "SimulatorConfig: c_neg must be < 0");
  if (c->n_interp < 0) return fail(EVSIM_GPU_INVALID_ARGUMENT, "SimulatorConfig: n_interp must be >= 0");
  if (c->contrast_mode == EVSIM_CONTRAST_LOG && c->method == EVSIM_METHOD_DIFFERENCE_INTERP)
    return fail(EVSIM_GPU_INVALID_ARGUMENT, "SimulatorConfig: difference_interp has no log contrast mode");
  if (c->contrast_mode == EVSIM_CONTRAST_LOG) {
    if (!(c->c_pos_log > 0.0f)) return fail(EVSIM_GPU_INVALID_ARGUMENT, "SimulatorConfig: c_pos_log must be > 0");
    if (!(c->c_neg_log < 0.0f)) return fail(EVSIM_GPU_INVALID_ARGUMENT, "SimulatorConfig: c_neg_log must be < 0");
  }
  return 0;
}

int evsim_oracle_create(const evsim_gpu_config* cfg, evsim_oracle_sim** out) {
  int rc = validate_cfg(cfg);
  if (rc) return rc;
  evsim_oracle_sim* s = (evsim_oracle_sim*)calloc(1, sizeof *s);
  s->cfg = *cfg;
  resolve_preset(cfg, &s->levels, &s->iters, &s->radius);
  rc = check_preset(s->levels, s->iters, s->radius);
  if (rc) { free(s); return rc; }
  evsim_oracle_log_lut(s->lut);
  *out = s;
  return 0;
}

void evsim_oracle_destroy(evsim_oracle_sim* s) {
  if (!s) return;
  free(s->prev); free(s->ref); free(s->pdiff); free(s->ev.v); free(s);
}

int evsim_oracle_reset(evsim_oracle_sim* s) {
  s->has_prev = 0;
  s->has_pdiff = 0;
  return 0;
}

const float* evsim_oracle_ref_state(const evsim_oracle_sim* s) {
  return (s->cfg.contrast_mode == EVSIM_CONTRAST_LOG && s->has_prev) ? s->ref : NULL;
}

static void select_points(const evsim_oracle_sim* s, const uint8_t* prev, const uint8_t* curr,
                          int w, int h, int32_t** pts, int64_t* M) {
  /* simulate.cpp:149-159; log mode: |L(curr) - L(prev)| > sel_log */
  const evsim_gpu_config* c = &s->cfg;
  int64_t cap = 1024, n = 0;
  int32_t* p = (int32_t*)malloc((size_t)cap * 2 * sizeof(int32_t));
  const int sel = c->selection_threshold > 0 ? c->selection_threshold : c->c_pos;
  const float sel_log = c->sel_log > 0.0f ? c->sel_log : c->c_pos_log;
  for (int y = 0; y < h; ++y) {
    for (int x = 0; x < w; ++x) {
      const size_t i = (size_t)y * w + x;
      int take;
      if (c->contrast_mode == EVSIM_CONTRAST_LOG) take = fabsf(s->lut[curr[i]] - s->lut[prev[i]]) > sel_log;
      else take = abs((int)curr[i] - (int)prev[i]) > sel;
      if (take) {
        if (n == cap) { cap *= 2; p = (int32_t*)realloc(p, (size_t)cap * 2 * sizeof(int32_t)); }
        p[2 * n] = x;
        p[2 * n + 1] = y;
        ++n;
      }
    }
  }
  *pts = p;
  *M = n;
}

int evsim_oracle_push_frame(evsim_oracle_sim* s, const uint8_t* pixels, int32_t w, int32_t h,
                            int64_t t, const evsim_event** events, int64_t* n_events) {
  if (w <= 0 || h <= 0 || !pixels) return fail(EVSIM_GPU_INVALID_ARGUMENT, "push_frame: malformed frame");
  if (s->has_prev) {
    if (w != s->w || h != s->h)
      return fail(EVSIM_GPU_INVALID_ARGUMENT, "push_frame: frame dimensions changed mid-stream");
    if (t <= s->prev_t)
      return fail(EVSIM_GPU_INVALID_ARGUMENT, "push_frame: timestamps must be strictly increasing");
  }
  const size_t P = (size_t)w * h;
  s->ev.n = 0;
  chain_ctx cx = {&s->cfg, s->lut, s->ref};
  if (s->has_prev) {
    const uint8_t* prev = s->prev;
    switch (s->cfg.method) {
      case EVSIM_METHOD_DIFFERENCE_ONLY:
        /* simulate.cpp:322-327: one link, no finalize (already ordered) */
        link_events(&cx, prev, pixels, w, h, t, &s->ev);
        break;
      case EVSIM_METHOD_DENSE:
        if (s->cfg.n_interp == 0) {
          chain_pipeline(&cx, prev, s->prev_t, pixels, t, NULL, NULL, 0, w, h, &s->ev);
        } else {
          float* du = (float*)malloc(P * sizeof(float));
          float* dv = (float*)malloc(P * sizeof(float));
          evsim_oracle_dense_flow(prev, pixels, w, h, s->levels, s->iters, s->radius, du, dv);
          dense_with_flow(&cx, prev, pixels, w, h, s->prev_t, t, du, dv, &s->ev);
          free(du); free(dv);
        }
        break;
      case EVSIM_METHOD_SPARSE: {
        int32_t* pts;
        int64_t M;
        select_points(s, prev, pixels, w, h, &pts, &M);
        if (M == 0 || s->cfg.n_interp == 0) {
          chain_pipeline(&cx, prev, s->prev_t, pixels, t, NULL, NULL, 0, w, h, &s->ev);
        } else {
          float* disp = (float*)malloc((size_t)M * 2 * sizeof(float));
          uint8_t* st = (uint8_t*)malloc((size_t)M);
          evsim_oracle_sparse_flow(prev, pixels, w, h, s->levels, s->iters, s->radius, pts, M, disp, st);
          sparse_with_flow(&cx, prev, pixels, w, h, s->prev_t, t, pts, M, disp, st, &s->ev);
          free(disp); free(st);
        }
        free(pts);
        break;
      }
      case EVSIM_METHOD_DIFFERENCE_INTERP: {
        /* simulate.cpp:334-341: events need the previous difference frame */
        int16_t* d = (int16_t*)malloc(P * sizeof(int16_t));
        for (size_t i = 0; i < P; ++i) d[i] = (int16_t)((int)pixels[i] - (int)prev[i]);
        if (s->has_pdiff)
          diff_interp_events(&s->cfg, s->levels, s->iters, s->radius, s->pdiff, d, w, h, s->prev_t, t, &s->ev);
        free(s->pdiff);
        s->pdiff = d;
        s->has_pdiff = 1;
        break;
      }
    }
  }
  if (!s->has_prev || s->w != w || s->h != h) {
    free(s->prev);
    free(s->ref);
    s->prev = (uint8_t*)malloc(P);
    s->ref = (float*)malloc(P * sizeof(float));
  }
  if (!s->has_prev && s->cfg.contrast_mode == EVSIM_CONTRAST_LOG) {
    for (size_t i = 0; i < P; ++i) s->ref[i] = s->lut[pixels[i]]; /* ref := L(frame0) */
  }
  memcpy(s->prev, pixels, P);
  s->w = w;
  s->h = h;
  s->prev_t = t;
  s->has_prev = 1;
  *events = s->ev.v;
  *n_events = s->ev.n;
  return 0;
}

static int stateless_cfg(const evsim_gpu_config* cfg, chain_ctx* cx, float* lut) {
  int rc = validate_cfg(cfg);
  if (rc) return rc;
  if (cfg->contrast_mode != EVSIM_CONTRAST_LINEAR)
    return fail(EVSIM_GPU_INVALID_ARGUMENT, "events_with_flow: stateless entry points are linear-mode only");
  evsim_oracle_log_lut(lut);
  cx->cfg = cfg;
  cx->lut = lut;
  cx->ref = NULL;
  return 0;
}

int evsim_oracle_dense_events_with_flow(const uint8_t* prev, const uint8_t* curr, int32_t w,
                                        int32_t h, int64_t t_prev, int64_t t_curr,
                                        const float* du, const float* dv,
                                        const evsim_gpu_config* cfg, evsim_event** events,
                                        int64_t* n_events) {
  float lut[256];
  chain_ctx cx;
  int rc = stateless_cfg(cfg, &cx, lut);
  if (rc) return rc;
  evvec ev = {0};
  dense_with_flow(&cx, prev, curr, w, h, t_prev, t_curr, du, dv, &ev);
  *events = ev.v;
  *n_events = ev.n;
  return 0;
}

int evsim_oracle_sparse_events_with_flow(const uint8_t* prev, const uint8_t* curr, int32_t w,
                                         int32_t h, int64_t t_prev, int64_t t_curr,
                                         const int32_t* pts, int64_t M, const float* disp,
                                         const uint8_t* status, const evsim_gpu_config* cfg,
                                         evsim_event** events, int64_t* n_events) {
  float lut[256];
  chain_ctx cx;
  int rc = stateless_cfg(cfg, &cx, lut);
  if (rc) return rc;
  evvec ev = {0};
  if (M == 0 || cfg->n_interp == 0)
    chain_pipeline(&cx, prev, t_prev, curr, t_curr, NULL, NULL, 0, w, h, &ev);
  else
    sparse_with_flow(&cx, prev, curr, w, h, t_prev, t_curr, pts, M, disp, status, &ev);
  *events = ev.v;
  *n_events = ev.n;
  return 0;
}

void evsim_oracle_free(void* p) { free(p); }
