// Microbenchmark: MUFU.EX2 and FFMA throughput per SM per clock on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void ex2_kernel(float* out, int iters, long long* cyc) {
  float a[8];
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3f + k * 1e-4f;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[k]));
  }
  long long t1 = clock64();
  float s = 0; for (int k = 0; k < 8; ++k) s += a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
__global__ void ffma_kernel(float* out, int iters, long long* cyc) {
  float a[8];
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3f + k;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("fma.rn.f32 %0, %0, 0.999, 0.001;" : "+f"(a[k]));
  }
  long long t1 = clock64();
  float s = 0; for (int k = 0; k < 8; ++k) s += a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 8 * 4); cudaMallocManaged(&cyc, 8);
  const int iters = 4096;
  for (int threads : {128, 256, 512, 1024}) {
    for (int which = 0; which < 2; ++which) {
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      auto launch = [&] { if (which == 0) ex2_kernel<<<sms, threads>>>(out, iters, cyc); else ffma_kernel<<<sms, threads>>>(out, iters, cyc); };
      launch(); cudaDeviceSynchronize();
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops_per_sm = (double)threads * iters * 8;
      printf("%s threads/SM=%4d: %.2f ops/clk/SM (clock64 in CTA0: %lld cycles), %.3f ms\n", which ? "FFMA" : "EX2 ", threads,
             ops_per_sm / (double)*cyc, *cyc, ms);
    }
  }
  return 0;
}
