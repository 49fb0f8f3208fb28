// Microbenchmark: dependent-chain latency (cycles/op) of the FP ops on the
// LK critical path, on the B200.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void chain(double* out, float* outf, long long* cyc, int n, double seed, float fseed) {
  double a = seed, b = seed * 1.0000001;
  float f = fseed, g = fseed * 1.0001f;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (OP == 0) a = __dadd_rn(a, b);                       // DADD
    if (OP == 1) a = __dmul_rn(a, b);                       // DMUL
    if (OP == 2) f = __fadd_rn(f, g);                       // FADD
    if (OP == 3) { a = __dadd_rn(a, (double)f); f = __fadd_rn(f, g); }  // F2F feeding DADD
    if (OP == 4) a = __dadd_rn(a, (double)__int_as_float(__double2hiint(a) & 0x3f000000));  // F2F on path
    if (OP == 5) a = __fma_rn(a, b, b);                     // DFMA
  }
  long long t1 = clock64();
  out[0] = a; outf[0] = f; cyc[0] = t1 - t0;
}

__global__ void tput(double* out, long long* cyc, int n) {
  double a[8];
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x + j;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = __dadd_rn(a[j], 1.0000001);
  long long t1 = clock64();
  double s = 0; for (int j = 0; j < 8; ++j) s += a[j];
  out[threadIdx.x + blockIdx.x * blockDim.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* d; float* f; long long* c; cudaMalloc(&d, 1 << 24); cudaMalloc(&f, 64); cudaMalloc(&c, 64);
  const int n = 100000;
  const char* names[] = {"DADD", "DMUL", "FADD", "F2F+DADD", "F2F-on-path", "DFMA"};
  for (int op = 0; op < 6; ++op) {
    long long h = 0;
    for (int rep = 0; rep < 2; ++rep) {
      switch (op) {
        case 0: chain<0><<<1, 1>>>(d, f, c, n, 1.0, 1.0f); break;
        case 1: chain<1><<<1, 1>>>(d, f, c, n, 1.0, 1.0f); break;
        case 2: chain<2><<<1, 1>>>(d, f, c, n, 1.0, 1.0f); break;
        case 3: chain<3><<<1, 1>>>(d, f, c, n, 1.0, 1.0f); break;
        case 4: chain<4><<<1, 1>>>(d, f, c, n, 1.0, 1.0f); break;
        case 5: chain<5><<<1, 1>>>(d, f, c, n, 1.0, 1.0f); break;
      }
      cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    }
    printf("%-12s latency %.2f cycles/op\n", names[op], (double)h / n);
  }
  // throughput: 148*4 warps x 8 independent chains
  long long h = 0;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int m = 20000;
  tput<<<148 * 8, 256>>>(d, c, m);
  cudaEventRecord(e0);
  tput<<<148 * 8, 256>>>(d, c, m);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  const double ops = 148.0 * 8 * 256 * m * 8;
  printf("DADD throughput: %.1f Gop/s (%.2f ms)\n", ops / ms / 1e6, ms);
  return 0;
}
