// Probe: 3-D fp32 TMA box loads (no swizzle) into shared memory, as used by the
// TMA tile gather.  Prints per-case status; each case in its own process so an
// illegal instruction does not poison the others.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void k3(const __grid_constant__ CUtensorMap tm, float* out, int n, int x0, int y0, int z0, int use3d) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned long long* bar = (unsigned long long*)(sm + ((n * 4 + 15) & ~15));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(n * 4));
    if (use3d)
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                   ::"r"(su32(sm)), "l"((unsigned long long)&tm), "r"(su32(bar)), "r"(x0), "r"(y0), "r"(z0) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                   ::"r"(su32(sm)), "l"((unsigned long long)&tm), "r"(su32(bar)), "r"(x0), "r"(y0) : "memory");
  }
  unsigned ok = 0;
  while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(bar)));
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = ((float*)sm)[i];
}
int main(int argc, char** argv) {
  int W = atoi(argv[1]), H = atoi(argv[2]), Z = atoi(argv[3]), b0 = atoi(argv[4]), b1 = atoi(argv[5]), b2 = atoi(argv[6]);
  int x0 = atoi(argv[7]), y0 = atoi(argv[8]), z0 = atoi(argv[9]), use3d = atoi(argv[10]);
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  std::vector<float> h((size_t)W * H * Z);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
  float *d, *o; cudaMalloc(&d, h.size() * 4); cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  int n = use3d ? b0 * b1 * b2 : b0 * b1;
  cudaMalloc(&o, n * 4);
  CUtensorMap tm;
  cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)Z};
  cuuint64_t str[2] = {(cuuint64_t)W * 4, (cuuint64_t)W * H * 4};
  cuuint32_t box[3] = {(cuuint32_t)b0, (cuuint32_t)b1, (cuuint32_t)b2}, es[3] = {1, 1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, use3d ? 3 : 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  int smem = ((n * 4 + 15) & ~15) + 16;
  cudaFuncSetAttribute(k3, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k3<<<1, 128, smem>>>(tm, o, n, x0, y0, z0, use3d);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> ho(n); cudaMemcpy(ho.data(), o, n * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int k = 0; k < (use3d ? b2 : 1); ++k) for (int j = 0; j < b1; ++j) for (int i = 0; i < b0; ++i) {
    int X = x0 + i, Y = y0 + j, Zz = z0 + k;
    float want = (X < W && Y < H && Zz < Z) ? (float)(((size_t)Zz * H + Y) * W + X) : 0.f;
    if (ho[((size_t)k * b1 + j) * b0 + i] != want) ++bad;
  }
  printf("W=%d H=%d Z=%d box %d %d %d at %d %d %d 3d=%d: %s, mismatches %d\n", W, H, Z, b0, b1, b2, x0, y0, z0, use3d,
         cudaGetErrorString(e), bad);
  return 0;
}
