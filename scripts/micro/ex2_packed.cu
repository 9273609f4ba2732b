// Microbenchmark: packed half-precision exp2 (ex2.approx.f16x2 / .ftz.bf16x2)
// versus ex2.approx.ftz.f32: exponentials per clock per SM, and the SASS
// each compiles to.  8 independent chains per thread, 512 threads per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, int iters, long long* cyc) {
  uint32_t h[8];
  float f[8];
  for (int j = 0; j < 8; ++j) {
    h[j] = 0x3c003c00u ^ (threadIdx.x & 7);   // ~1.0 halves
    f[j] = threadIdx.x * 1e-3f + j * 1e-4f;
  }
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[j]));
      if (MODE == 1) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h[j]));
      if (MODE == 2) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h[j]));
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int j = 0; j < 8; ++j) s += f[j] + (float)h[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMallocManaged(&cyc, 8);
  const int iters = 4096, threads = 512;
  const char* names[3] = {"ex2.approx.ftz.f32    ", "ex2.approx.f16x2      ", "ex2.approx.ftz.bf16x2 "};
  for (int m = 0; m < 3; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      if (m == 0) k<0><<<sms, threads>>>(out, iters, cyc);
      if (m == 1) k<1><<<sms, threads>>>(out, iters, cyc);
      if (m == 2) k<2><<<sms, threads>>>(out, iters, cyc);
      cudaDeviceSynchronize();
    }
    const double instr = (double)threads * iters * 8;
    const double elems = instr * (m == 0 ? 1 : 2);
    printf("%s: %.2f instr/clk/SM, %.2f exps/clk/SM (%lld cycles)\n", names[m], instr / (double)*cyc,
           elems / (double)*cyc, *cyc);
  }
  return 0;
}
