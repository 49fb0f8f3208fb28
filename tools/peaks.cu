// peaks.cu — measured compute peaks of this B200 for the roofline of the
// CUDA-core kernels (the chain, the LK solver): FP32 FFMA, FP32x2 FFMA2,
// FP64 DADD / DFMA, the ALU pipe (LOP3), and the warp-instruction issue rate.
// Each kernel runs 8 independent accumulator chains per thread (enough ILP
// to hide the pipe latency), 148 x 8 blocks of 256 threads, timed with CUDA
// events after a warm-up; the result is the best of 5 runs.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/peaks tools/peaks.cu
//   tools/peaks > profiles/r02/peaks.json
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e = (x);                                                           \
    if (e != cudaSuccess) {                                                        \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

constexpr int kIters = 4096;
constexpr int kChains = 8;

__global__ void ffma_kernel(float* out, float a, float b) {
  float x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 0.001f + c;
  for (int i = 0; i < kIters; ++i)
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = __fmaf_rn(x[c], a, b);
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 1234.5f) out[0] = s;
}

__global__ void ffma2_kernel(float* out, float a, float b) {
  unsigned long long x[kChains];
  unsigned long long A, B;
  asm("mov.b64 %0, {%1, %1};" : "=l"(A) : "f"(a));
  asm("mov.b64 %0, {%1, %1};" : "=l"(B) : "f"(b));
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    const float v = threadIdx.x * 0.001f + c;
    asm("mov.b64 %0, {%1, %1};" : "=l"(x[c]) : "f"(v));
  }
  for (int i = 0; i < kIters; ++i)
#pragma unroll
    for (int c = 0; c < kChains; ++c) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[c]) : "l"(A), "l"(B));
  unsigned long long s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s ^= x[c];
  if (s == 12345ull) out[0] = 1.f;
}

__global__ void dadd_kernel(double* out, double a) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 0.001 + c;
  for (int i = 0; i < kIters; ++i)
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = __dadd_rn(x[c], a);
  double s = 0.;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 1234.5) out[0] = s;
}

__global__ void dfma_kernel(double* out, double a, double b) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 0.001 + c;
  for (int i = 0; i < kIters; ++i)
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = __fma_rn(x[c], a, b);
  double s = 0.;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 1234.5) out[0] = s;
}

__global__ void lop3_kernel(unsigned* out, unsigned a, unsigned b) {
  unsigned x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 2654435761u + c;
  for (int i = 0; i < kIters; ++i)
#pragma unroll
    for (int c = 0; c < kChains; ++c) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(a), "r"(b));
  unsigned s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s ^= x[c];
  if (s == 12345u) out[0] = s;
}

// alternating fma-pipe and alu-pipe instructions: the issue ceiling of a mix
__global__ void mix_kernel(float* out, float a, float b, unsigned ua, unsigned ub) {
  float x[kChains / 2];
  unsigned y[kChains / 2];
#pragma unroll
  for (int c = 0; c < kChains / 2; ++c) x[c] = threadIdx.x * 0.001f + c, y[c] = threadIdx.x + c;
  for (int i = 0; i < kIters; ++i)
#pragma unroll
    for (int c = 0; c < kChains / 2; ++c) {
      x[c] = __fmaf_rn(x[c], a, b);
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(y[c]) : "r"(ua), "r"(ub));
    }
  float s = 0.f;
  unsigned t = 0;
#pragma unroll
  for (int c = 0; c < kChains / 2; ++c) s += x[c], t ^= y[c];
  if (s == 1234.5f || t == 7u) out[0] = s;
}

template <class F>
float best_ms(F launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return best;
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const int sms = prop.multiProcessorCount;
  const dim3 grid(sms * 8), block(256);
  float* f;
  double* d;
  unsigned* u;
  CK(cudaMalloc(&f, 64));
  CK(cudaMalloc(&d, 64));
  CK(cudaMalloc(&u, 64));
  const double threads = (double)grid.x * block.x;
  const double ops = threads * kIters * kChains;       // instructions per thread x threads
  const double warp_instr = ops / 32.0;                // warp-instructions of the timed loop
  const float t_ffma = best_ms([&] { ffma_kernel<<<grid, block>>>(f, 0.999f, 0.001f); });
  const float t_ffma2 = best_ms([&] { ffma2_kernel<<<grid, block>>>(f, 0.999f, 0.001f); });
  const float t_dadd = best_ms([&] { dadd_kernel<<<grid, block>>>(d, 1e-9); });
  const float t_dfma = best_ms([&] { dfma_kernel<<<grid, block>>>(d, 0.999, 0.001); });
  const float t_lop3 = best_ms([&] { lop3_kernel<<<grid, block>>>(u, 0x5bd1e995u, 0x1b873593u); });
  const float t_mix = best_ms([&] { mix_kernel<<<grid, block>>>(f, 0.999f, 0.001f, 0x5bd1e995u, 0x1b873593u); });
  CK(cudaGetLastError());
  auto tf = [&](float ms, double flops_per_op) { return ops * flops_per_op / (ms * 1e-3) / 1e12; };
  auto gi = [&](float ms) { return warp_instr / (ms * 1e-3) / 1e9; };
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_mhz_attr\": %.0f,\n", prop.name, sms, clk_khz / 1e3);
  printf(" \"fp32_ffma_tflops\": %.2f, \"fp32x2_ffma2_tflops\": %.2f, \"fp64_dadd_tflops\": %.3f, "
         "\"fp64_dfma_tflops\": %.3f,\n",
         tf(t_ffma, 2), tf(t_ffma2, 4), tf(t_dadd, 1), tf(t_dfma, 2));
  printf(" \"warp_instr_per_s_G\": {\"ffma\": %.1f, \"ffma2\": %.1f, \"dadd\": %.1f, \"dfma\": %.1f, \"lop3\": %.1f, "
         "\"ffma+lop3\": %.1f},\n",
         gi(t_ffma), gi(t_ffma2), gi(t_dadd), gi(t_dfma), gi(t_lop3), gi(t_mix));
  printf(" \"issue_peak_G_per_s_theoretical\": %.1f,\n", sms * 4.0 * clk_khz / 1e6);
  printf(" \"how\": \"%d blocks x 256 threads, %d iterations x %d independent chains per thread, best of 5 "
         "(CUDA events); tools/peaks.cu\"}\n",
         grid.x, kIters, kChains);
  return 0;
}
