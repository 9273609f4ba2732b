// Microbenchmark: the attention softmax exp loop in isolation.
// Each thread holds NE S values in registers and repeatedly computes
// p = 2^(s*c - m) (FFMA2 + MUFU.EX2), packs pairs to bf16 (F2FP) and sums
// (FADD), exactly as attn_tc.cu does per 128-key block.  m is re-read from
// shared memory every round so nothing is hoisted.  Reports cycles per round
// for 1, 2 and 4 warps per SM sub-partition (128/256/512 threads per SM).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void ffma2(float& a, float& b, float s, float t) {
  asm("{\n\t.reg .b64 x, sc, tt;\n\tmov.b64 x, {%0, %1};\n\tmov.b64 sc, {%2, %2};\n\t"
      "mov.b64 tt, {%3, %3};\n\tfma.rn.f32x2 x, x, sc, tt;\n\tmov.b64 {%0, %1}, x;\n\t}"
      : "+f"(a), "+f"(b) : "f"(s), "f"(t));
}
__device__ __forceinline__ uint32_t pack(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

template <int NE, int MODE>   // MODE 0: full loop; 1: no pack; 2: no sum; 3: ex2 only
__global__ void k(const float* in, float* out, int rounds, long long* cyc) {
  __shared__ float m_sh[1];
  if (threadIdx.x == 0) m_sh[0] = 0.5f;
  __syncthreads();
  float sv[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) sv[e] = in[(threadIdx.x * NE + e) & 4095];
  uint32_t acc = 0;
  float l = 0.f;
  long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    float z;
    asm volatile("ld.volatile.shared.f32 %0, [%1];" : "=f"(z) : "r"((uint32_t)__cvta_generic_to_shared(m_sh)) : "memory");
    const float m = z + (float)r * 1e-7f;
    float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
    for (int e = 0; e < NE; e += 2) {
      float x0 = sv[e], x1 = sv[e + 1];
      if (MODE != 3) ffma2(x0, x1, 0.18f, -m);
      const float p0 = ex2(x0), p1 = ex2(x1);
      if (MODE != 2 && MODE != 3) { rs0 += p0; rs1 += p1; }
      if (MODE != 1 && MODE != 3) acc ^= pack(p0, p1);
      if (MODE == 3) acc ^= __float_as_uint(p0) ^ __float_as_uint(p1);
    }
    l += rs0 + rs1;
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = l + (float)acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *in, *out;
  long long* cyc;
  cudaMalloc(&in, 4096 * 4);
  cudaMemset(in, 0, 4096 * 4);
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMallocManaged(&cyc, 8);
  const int rounds = 256;
  const char* mn[4] = {"full (ffma2+ex2+pack+sum)", "no pack", "no sum", "ex2 only"};
  for (int mode = 0; mode < 4; ++mode)
    for (int threads : {128, 256, 512}) {
      for (int ne : {64, 128}) {
        auto launch = [&] {
          if (ne == 128) {
            if (mode == 0) k<128, 0><<<sms, threads>>>(in, out, rounds, cyc);
            if (mode == 1) k<128, 1><<<sms, threads>>>(in, out, rounds, cyc);
            if (mode == 2) k<128, 2><<<sms, threads>>>(in, out, rounds, cyc);
            if (mode == 3) k<128, 3><<<sms, threads>>>(in, out, rounds, cyc);
          } else {
            if (mode == 0) k<64, 0><<<sms, threads>>>(in, out, rounds, cyc);
            if (mode == 1) k<64, 1><<<sms, threads>>>(in, out, rounds, cyc);
            if (mode == 2) k<64, 2><<<sms, threads>>>(in, out, rounds, cyc);
            if (mode == 3) k<64, 3><<<sms, threads>>>(in, out, rounds, cyc);
          }
        };
        launch();
        cudaDeviceSynchronize();
        launch();
        cudaDeviceSynchronize();
        const double ex_per_sm = (double)threads * ne * rounds;
        printf("%-26s warps/SMSP=%d NE=%3d: %.2f ex2/clk/SM, %.0f cycles per 16384 exps\n", mn[mode], threads / 128, ne,
               ex_per_sm / (double)*cyc, 16384.0 * (double)*cyc / ex_per_sm);
      }
    }
  return 0;
}
