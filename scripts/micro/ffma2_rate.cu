// Microbenchmark: FFMA vs packed FFMA2 (fma.rn.f32x2) / FMUL2 throughput on sm_100a.
// 8 independent chains per thread, 512 threads per SM.  Reports fp32 FMAs per
// clock per SM (an FFMA2 counts as 2).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, int iters, long long* cyc) {
  float a[16];
  for (int j = 0; j < 16; ++j) a[j] = threadIdx.x * 1e-3f + j;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; j += 2) {
      if (MODE == 0) {
        asm volatile("fma.rn.f32 %0, %0, 0f3F7FBE77, 0f3A83126F;" : "+f"(a[j]));
        asm volatile("fma.rn.f32 %0, %0, 0f3F7FBE77, 0f3A83126F;" : "+f"(a[j + 1]));
      } else if (MODE == 1) {
        asm volatile(
            "{\n\t.reg .b64 x, s, t;\n\tmov.b64 x, {%0, %1};\n\tmov.b64 s, {0f3F7FBE77, 0f3F7FBE77};\n\t"
            "mov.b64 t, {0f3A83126F, 0f3A83126F};\n\tfma.rn.f32x2 x, x, s, t;\n\tmov.b64 {%0, %1}, x;\n\t}"
            : "+f"(a[j]), "+f"(a[j + 1]));
      } else {
        asm volatile(
            "{\n\t.reg .b64 x, s;\n\tmov.b64 x, {%0, %1};\n\tmov.b64 s, {0f3F7FBE77, 0f3F7FBE77};\n\t"
            "mul.rn.f32x2 x, x, s;\n\tmov.b64 {%0, %1}, x;\n\t}"
            : "+f"(a[j]), "+f"(a[j + 1]));
      }
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int j = 0; j < 16; ++j) s += a[j];
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
  const int iters = 4096;
  const char* names[3] = {"FFMA  (fma.rn.f32)   ", "FFMA2 (fma.rn.f32x2) ", "FMUL2 (mul.rn.f32x2) "};
  for (int threads : {256, 512}) {
    for (int m = 0; m < 3; ++m) {
      for (int rep = 0; rep < 2; ++rep) {
        if (m == 0) k<0><<<sms, threads>>>(out, iters, cyc);
        if (m == 1) k<1><<<sms, threads>>>(out, iters, cyc);
        if (m == 2) k<2><<<sms, threads>>>(out, iters, cyc);
        cudaDeviceSynchronize();
      }
      const double flops = (double)threads * iters * 16;
      printf("threads/SM=%d %s: %.1f fp32 ops/clk/SM (%lld cycles)\n", threads, names[m], flops / (double)*cyc, *cyc);
    }
  }
  return 0;
}
