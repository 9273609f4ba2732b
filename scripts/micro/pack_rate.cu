// Microbenchmark: does the bf16 pack (F2FP.BF16.F32.PACK_AB) share the MUFU pipe?
// Kernels (8 independent chains per thread, 512 threads per SM):
//   ex2   : ex2.approx only
//   f2fp  : cvt.rn.bf16x2.f32 only
//   mix   : 2 ex2 + 1 cvt (the softmax inner-loop ratio)
//   mixi  : 2 ex2 + integer round/pack (2 IADD + PRMT)
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float* out, int iters, long long* cyc) {
  float a[8];
  unsigned u[8];
  for (int j = 0; j < 8; ++j) { a[j] = threadIdx.x * 1e-3f + j * 1e-4f; u[j] = j; }
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; j += 2) {
      if (MODE == 0 || MODE == 2 || MODE == 3) {
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[j]));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[j + 1]));
      }
      if (MODE == 1 || MODE == 2)
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u[j]) : "f"(a[j]), "f"(a[j + 1]));
      if (MODE == 1) asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u[j + 1]) : "f"(a[j + 1]), "f"(a[j]));
      if (MODE == 3) {
        unsigned x0 = __float_as_uint(a[j]) + 0x8000u, x1 = __float_as_uint(a[j + 1]) + 0x8000u;
        asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(u[j]) : "r"(x0), "r"(x1));
      }
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int j = 0; j < 8; ++j) s += a[j] + (float)u[j];
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
  const char* names[4] = {"ex2 only        ", "cvt.bf16x2 only ", "2 ex2 + 1 cvt   ", "2 ex2 + int pack"};
  for (int m = 0; m < 4; ++m) {
    auto launch = [&] {
      if (m == 0) k<0><<<sms, threads>>>(out, iters, cyc);
      if (m == 1) k<1><<<sms, threads>>>(out, iters, cyc);
      if (m == 2) k<2><<<sms, threads>>>(out, iters, cyc);
      if (m == 3) k<3><<<sms, threads>>>(out, iters, cyc);
    };
    launch();
    cudaDeviceSynchronize();
    launch();
    cudaDeviceSynchronize();
    // per thread: 8 elements per iteration (ex2 count for modes 0,2,3; cvt count for mode 1)
    double per_sm = (double)threads * iters * 8;
    printf("%s: %.2f elements/clk/SM (%lld cycles)\n", names[m], per_sm / (double)*cyc, *cyc);
  }
  return 0;
}
