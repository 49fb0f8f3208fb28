// evsim_device.cuh — bit-exact device arithmetic shared by the sm_100a kernels.
//
// The reference (C++, x86-64, SSE2 scalar, no FMA) fixes the rounding of every
// intermediate.  All kernels are compiled with -fmad=false and the helpers
// below spell out each rounding step with the _rn intrinsics so that nvcc can
// never contract or reassociate them.  Citations: /root/reference/proj/...
#pragma once

#include <cstdint>
#include <cstdio>

namespace evsim_gpu {

// Checked build (build.py --checked -> libevsim_gpu_checked.so, -DEVSIM_CHECKED):
// bounds checks of the kernels' global writes against their buffers' sizes
// and of the staging indices; a violation prints the site and traps (the
// context is lost, so the calling test fails loudly).  compute-sanitizer is
// not available on the GPU pool; tests/test_checked_build.py runs the GPU
// parity subset on this build instead.  Compiled out otherwise.
#ifdef EVSIM_CHECKED
#define EVSIM_CHECK(cond, what)                                                                            \
  do {                                                                                                     \
    if (!(cond)) {                                                                                         \
      printf("EVSIM_CHECKED: %s violated at %s:%d (block %d,%d,%d thread %d)\n", what, __FILE__, __LINE__, \
             (int)blockIdx.x, (int)blockIdx.y, (int)blockIdx.z, (int)threadIdx.x);                         \
      __trap();                                                                                            \
    }                                                                                                      \
  } while (0)
#else
#define EVSIM_CHECK(cond, what) \
  do {                          \
  } while (0)
#endif


constexpr unsigned kFull = 0xFFFFFFFFu;

// std::clamp(v, lo, hi) (lo if v < lo; hi if hi < v; else v — NaN passes through).
__device__ __forceinline__ float clamp_ref(float v, float lo, float hi) {
  return (v < lo) ? lo : ((hi < v) ? hi : v);
}
__device__ __forceinline__ int clampi(int v, int lo, int hi) { return (v < lo) ? lo : ((hi < v) ? hi : v); }

__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }

// Exact u8 -> float without the I2F pipe: 2^23 + b has b in the mantissa.
__device__ __forceinline__ float u8f(uint32_t b) {
  return __fsub_rn(__uint_as_float(0x4B000000u | b), 8388608.0f);
}

// lerp step used by every bilinear sample in the reference:
//   a + f * (b - a)   (flow.cpp:54-56, simulate.cpp:19-21)
__device__ __forceinline__ float lerp_ref(float a, float b, float f) { return fadd(a, fmul(f, fsub(b, a))); }

// Clamped coordinate split of sample()/sample_u8() (flow.cpp:46-53, simulate.cpp:11-18).
struct Tap {
  int x0, y0, x1, y1;
  float fx, fy;
};
__device__ __forceinline__ Tap make_tap(float x, float y, int w, int h) {
  x = clamp_ref(x, 0.0f, (float)(w - 1));
  y = clamp_ref(y, 0.0f, (float)(h - 1));
  Tap t;
  t.x0 = (int)x;  // truncation, x >= 0
  t.y0 = (int)y;
  t.x1 = min(t.x0 + 1, w - 1);
  t.y1 = min(t.y0 + 1, h - 1);
  t.fx = fsub(x, (float)t.x0);
  t.fy = fsub(y, (float)t.y0);
  return t;
}

// sample() over an fp32 image, flow.cpp:45-57.
__device__ __forceinline__ float sample_f32(const float* __restrict__ im, int w, int h, float x, float y) {
  const Tap t = make_tap(x, y, w, h);
  const float* r0 = im + (size_t)t.y0 * w;
  const float* r1 = im + (size_t)t.y1 * w;
  const float top = lerp_ref(__ldg(r0 + t.x0), __ldg(r0 + t.x1), t.fx);
  const float bot = lerp_ref(__ldg(r1 + t.x0), __ldg(r1 + t.x1), t.fx);
  return lerp_ref(top, bot, t.fy);
}

// sample_u8() (simulate.cpp:10-26) over a QUAD image: q[y*w+x] packs the four
// bilinear taps (x0,y0) (x1,y0) (x0,y1) (x1,y1) of the clamped neighbourhood
// in bytes 0..3, so one 32-bit gather replaces four byte gathers.
__device__ __forceinline__ float sample_quad(const uint32_t* __restrict__ q, int w, int h, float x, float y) {
  x = clamp_ref(x, 0.0f, (float)(w - 1));
  y = clamp_ref(y, 0.0f, (float)(h - 1));
  const int x0 = (int)x;
  const int y0 = (int)y;
  const float fx = fsub(x, (float)x0);
  const float fy = fsub(y, (float)y0);
  const uint32_t v = __ldg(q + (size_t)y0 * w + x0);
  const float a00 = u8f(v & 0xFFu);
  const float a10 = u8f((v >> 8) & 0xFFu);
  const float a01 = u8f((v >> 16) & 0xFFu);
  const float a11 = u8f(v >> 24);
  const float top = lerp_ref(a00, a10, fx);
  const float bot = lerp_ref(a01, a11, fx);
  return lerp_ref(top, bot, fy);
}

// ---- conversion-pipe-free variants (F2I/I2F/F2F run at 1/4 rate on sm_100) ----
// Valid for FINITE inputs only (the clamp uses FMNMX, which drops NaN); used
// where the coordinates come from our own (always finite) flow.

// trunc(x) for x in [0, 2^23): the RZ add leaves 2^23 + trunc(x) exactly.
__device__ __forceinline__ float trunc_magic(float x, int& xi) {
  const float t = __fadd_rz(x, 8388608.0f);
  xi = __float_as_int(t) - 0x4B000000;
  return __fsub_rn(t, 8388608.0f);
}

// byte k of v as an exact float: PRMT builds 0x4B0000bb, FADD removes 2^23.
template <int kByte>
__device__ __forceinline__ float byte_f(uint32_t v) {
  return __fsub_rn(__uint_as_float(__byte_perm(v, 0x4B000000u, 0x7540 + kByte)), 8388608.0f);
}

// sample_u8 through a quad image, finite coordinates (simulate.cpp:10-26).
__device__ __forceinline__ float sample_quad_fast(const uint32_t* __restrict__ q, int w, int h, float x, float y) {
  x = fminf(fmaxf(x, 0.0f), (float)(w - 1));
  y = fminf(fmaxf(y, 0.0f), (float)(h - 1));
  int x0, y0;
  const float x0f = trunc_magic(x, x0);
  const float y0f = trunc_magic(y, y0);
  const float fx = fsub(x, x0f);
  const float fy = fsub(y, y0f);
  const uint32_t v = __ldg(q + (size_t)y0 * w + x0);
  const float top = lerp_ref(byte_f<0>(v), byte_f<1>(v), fx);
  const float bot = lerp_ref(byte_f<2>(v), byte_f<3>(v), fx);
  return lerp_ref(top, bot, fy);
}

// ---- register pinning and 32-bit shared addressing for hot loops ----
// A value passed through a shuffle cannot be rematerialised by ptxas, so a
// ring base pointer or a constant used in a loop stays in one register
// instead of being recomputed (64-bit folding, immediate moves) per use.
template <typename T>
__device__ __forceinline__ T pin(T v) {
  static_assert(sizeof(T) == 4 || sizeof(T) == 8, "pin: 32- or 64-bit values");
  if constexpr (sizeof(T) == 8) {
    unsigned long long u;
    memcpy(&u, &v, 8);
    u = __shfl_sync(0xFFFFFFFFu, u, 0);
    memcpy(&v, &u, 8);
  } else {
    unsigned u;
    memcpy(&u, &v, 4);
    u = __shfl_sync(0xFFFFFFFFu, u, 0);
    memcpy(&v, &u, 4);
  }
  return v;
}
// ld.shared.f32 [a + kOff] (a: a shared-window byte address)
template <int kOff>
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(a), "n"(kOff));
  return v;
}

// ---- packed fp32x2 (sm_100 FADD2 / FMUL2): two independent IEEE fp32 ops per
// instruction, each lane rounded exactly like its scalar counterpart ----
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pk2(float lo, float hi) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float lo2(f32x2 v) {
  float lo;
  asm("{.reg .f32 t; mov.b64 {%0, t}, %1;}" : "=f"(lo) : "l"(v));
  return lo;
}
__device__ __forceinline__ float hi2(f32x2 v) {
  float hi;
  asm("{.reg .f32 t; mov.b64 {t, %0}, %1;}" : "=f"(hi) : "l"(v));
  return hi;
}
__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2 sub2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2 add2_rz(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("add.rz.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
// a + f * (b - a) on both lanes (the reference's lerp, flow.cpp:54-56).
// CAUTION: ptxas (CUDA 12.9) contracts mul.rn.f32x2 + add.rn.f32x2 into FFMA2
// even with --fmad=false, which would drop the reference's intermediate
// rounding.  The final adds are therefore scalar __fadd_rn (never fused).
__device__ __forceinline__ f32x2 lerp2(f32x2 a, f32x2 b, f32x2 f) {
  const f32x2 m = mul2(f, sub2(b, a));
  return pk2(__fadd_rn(lo2(a), lo2(m)), __fadd_rn(hi2(a), hi2(m)));
}
// a + f * d on both lanes, d = b - a already formed (exactly) by the caller
__device__ __forceinline__ f32x2 lerpd2(f32x2 a, f32x2 d, f32x2 f) {
  const f32x2 m = mul2(f, d);
  return pk2(__fadd_rn(lo2(a), lo2(m)), __fadd_rn(hi2(a), hi2(m)));
}
// (c + s*u, c + t*u) for s, t = lanes of st, as the reference's separate mul + add
__device__ __forceinline__ f32x2 affine2(float c, f32x2 st, float u) {
  const f32x2 m = mul2(st, pk2(u, u));
  return pk2(__fadd_rn(c, lo2(m)), __fadd_rn(c, hi2(m)));
}

// Estimate-only variants (dense_fast): the final adds as one FADD2.FTZ —
// ptxas does not contract mul.f32x2 into add.ftz.f32x2.  Flushing a denormal
// input / result moves a sample by < 255 * 2^-126, far inside the bounded
// estimate's 2e-4 decision margin, so a decided lane is unaffected; these
// must not be used where a result has to be exact.
__device__ __forceinline__ f32x2 add2_ftz(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("add.rn.ftz.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2 lerp2_est(f32x2 a, f32x2 b, f32x2 f) { return add2_ftz(a, mul2(f, sub2(b, a))); }
__device__ __forceinline__ f32x2 lerpd2_est(f32x2 a, f32x2 d, f32x2 f) { return add2_ftz(a, mul2(f, d)); }
__device__ __forceinline__ f32x2 affine2_est(float c, f32x2 st, float u) {
  return add2_ftz(pk2(c, c), mul2(st, pk2(u, u)));
}

// Two sample_u8 (simulate.cpp:10-26) through quad images at once: lane 0 =
// (x.lo, y.lo) in qa, lane 1 = (x.hi, y.hi) in qb.  Finite coordinates only.
__device__ __forceinline__ f32x2 sample_quad_pair(const uint32_t* __restrict__ qa, const uint32_t* __restrict__ qb,
                                                  int w, int h, f32x2 x, f32x2 y) {
  const float wm = (float)(w - 1), hm = (float)(h - 1);
  const f32x2 X = pk2(fminf(fmaxf(lo2(x), 0.0f), wm), fminf(fmaxf(hi2(x), 0.0f), wm));
  const f32x2 Y = pk2(fminf(fmaxf(lo2(y), 0.0f), hm), fminf(fmaxf(hi2(y), 0.0f), hm));
  const f32x2 C23 = pk2(8388608.0f, 8388608.0f);
  const f32x2 TX = add2_rz(X, C23), TY = add2_rz(Y, C23);  // 2^23 + trunc
  const int xa = __float_as_int(lo2(TX)) - 0x4B000000, xb = __float_as_int(hi2(TX)) - 0x4B000000;
  const int ya = __float_as_int(lo2(TY)) - 0x4B000000, yb = __float_as_int(hi2(TY)) - 0x4B000000;
  const f32x2 FX = sub2(X, sub2(TX, C23));
  const f32x2 FY = sub2(Y, sub2(TY, C23));
  const uint32_t va = __ldg(qa + (size_t)ya * w + xa);
  const uint32_t vb = __ldg(qb + (size_t)yb * w + xb);
  // bytes -> 2^23 + b (PRMT), minus 2^23 (exact)
  const f32x2 A00 = sub2(pk2(__uint_as_float(__byte_perm(va, 0x4B000000u, 0x7540)),
                             __uint_as_float(__byte_perm(vb, 0x4B000000u, 0x7540))), C23);
  const f32x2 A10 = sub2(pk2(__uint_as_float(__byte_perm(va, 0x4B000000u, 0x7541)),
                             __uint_as_float(__byte_perm(vb, 0x4B000000u, 0x7541))), C23);
  const f32x2 A01 = sub2(pk2(__uint_as_float(__byte_perm(va, 0x4B000000u, 0x7542)),
                             __uint_as_float(__byte_perm(vb, 0x4B000000u, 0x7542))), C23);
  const f32x2 A11 = sub2(pk2(__uint_as_float(__byte_perm(va, 0x4B000000u, 0x7543)),
                             __uint_as_float(__byte_perm(vb, 0x4B000000u, 0x7543))), C23);
  return lerp2(lerp2(A00, A10, FX), lerp2(A01, A11, FX), FY);
}

// lround() of v in [0, 2^31) without conversions: t = 2^52 + trunc(v) (RZ),
// its low word is trunc(v); v - trunc(v) is exact.
__device__ __forceinline__ int lround_pos_fast(double v) {
  const double t = __dadd_rz(v, 4503599627370496.0);
  const double f = __dsub_rn(t, 4503599627370496.0);
  return __double2loint(t) + ((__dsub_rn(v, f) >= 0.5) ? 1 : 0);
}

// lround() for a non-negative double (simulate.cpp:114): half away from zero.
// v - floor(v) is exact, so the comparison with 0.5 is exact.
__device__ __forceinline__ int lround_pos(double v) {
  const double f = floor(v);
  return (int)f + ((v - f) >= 0.5 ? 1 : 0);
}

// lroundf() for any float (simulate.cpp:181-184).
__device__ __forceinline__ int lroundf_ref(float v) {
  const float t = truncf(v);
  const float d = fsub(v, t);  // exact
  if (d >= 0.5f) return (int)t + 1;
  if (d <= -0.5f) return (int)t - 1;
  return (int)t;
}

// min_eigenvalue  flow.cpp:89-93
__device__ __forceinline__ double min_eigenvalue(double gxx, double gxy, double gyy) {
  const double trace = dadd(gxx, gyy);
  const double a = dsub(gxx, gyy);
  const double dd = dadd(dmul(a, a), dmul(dmul(4.0, gxy), gxy));
  const double disc = __dsqrt_rn(dd > 0.0 ? dd : 0.0);
  return dmul(0.5, dsub(trace, disc));
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

}  // namespace evsim_gpu
