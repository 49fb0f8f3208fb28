// evsim_device.cuh — bit-exact device arithmetic shared by the sm_100a kernels.
//
// The reference (C++, x86-64, SSE2 scalar, no FMA) fixes the rounding of every
// intermediate.  All kernels are compiled with -fmad=false and the helpers
// below spell out each rounding step with the _rn intrinsics so that nvcc can
// never contract or reassociate them.  Citations: /root/reference/proj/...
#pragma once

#include <cstdint>

namespace evsim_gpu {

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
