// rconv.cu -- steps (4)-(5) with the residual convolutional path (reading
// R31): crop + stitch + residual, where the residual is
//     res = up + conv_b(GELU(conv_a(up)))
// up = the bilinear x s upsample of the mapped input channels (O7), conv_a: 3x3,
// K -> C_r channels, conv_b: 3x3, C_r -> K, zero padding outside the
// high-resolution field.  The residual is a function of the input field only, so
// every output pixel is computed from x directly -- no dependence on other tiles'
// outputs (with halo >= 1 patch the padded rectangle holds the 2-output-pixel
// receptive field: TILES-consistent, oracle O8).
//
// One CTA per (output block of P rows x BX columns inside a tile's core, tile,
// sample): up on the block grown by 2 pixels -> shared memory; hidden layer
// GELU(conv_a(up)) on the block grown by 1 -> shared memory; conv_b + up + the
// decoder output (tile_out) -> out.  fp32 FMA on the CUDA cores (the C_r x K x 9
// contractions are 27-144 long per pixel); the weights are staged in shared memory.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>

#include "kernels.h"

namespace orbit2 {

namespace {

constexpr int BX = 64;          // output columns per CTA
constexpr int RC_THREADS = 256;

template <typename T> __device__ __forceinline__ float ld_f32(const T* p);
template <> __device__ __forceinline__ float ld_f32<float>(const float* p) { return *p; }
template <> __device__ __forceinline__ float ld_f32<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(*p);
}

__device__ __forceinline__ float gelu_exact(float x) { return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f)); }

template <typename T>
__global__ void __launch_bounds__(RC_THREADS) stitch_rconv_kernel(
    const T* __restrict__ tile_out, const float* __restrict__ x, float* __restrict__ out, ChunkDev ch,
    const int32_t* __restrict__ cmap, const float* __restrict__ wconv, int V, int H, int W, int K, int s, int P,
    int CR, int nseg) {
  extern __shared__ __align__(16) float rsm[];
  const int BY = P;
  const int UY = BY + 4, UX = BX + 4;               // up block (grown by 2)
  const int HY = BY + 2, HX = BX + 2;               // hidden block (grown by 1)
  float* sWa = rsm;                                 // [CR][K][9]
  float* sBa = sWa + CR * K * 9;                    // [CR]
  float* sWb = sBa + CR;                            // [K][CR][9]
  float* sBb = sWb + K * CR * 9;                    // [K]
  float* su = sBb + K;                              // [K][UY][UX]
  float* sh = su + K * UY * UX;                     // [CR][HY][HX]
  const DevTile t = ch.tiles[ch.tb + blockIdx.y];
  const int ur = blockIdx.x / nseg, seg = blockIdx.x - ur * nseg;
  if (ur >= t.core_h || seg * BX >= t.core_w * P) return;
  const int b = blockIdx.z;
  const int Y0 = (t.core_y0 + ur) * P;
  const int X0 = t.core_x0 * P + seg * BX;
  const int nx = min(BX, t.core_w * P - seg * BX);  // valid output columns of the block
  const int sH = s * H, sW = s * W;
  const int tid = threadIdx.x;
  const int nw = CR * K * 9 * 2 + CR + K;
  for (int i = tid; i < nw; i += RC_THREADS) rsm[i] = wconv[i];
  // up on the grown block (0 outside the field: conv_a's zero padding)
  const float inv_s = 1.0f / (float)s;
  for (int i = tid; i < K * UY * UX; i += RC_THREADS) {
    const int k = i / (UY * UX), r = i - k * UY * UX, yy = r / UX, xx = r - yy * UX;
    const int Y = Y0 - 2 + yy, X = X0 - 2 + xx;
    float v = 0.f;
    if (Y >= 0 && Y < sH && X >= 0 && X < sW) {
      const float sy = fmaxf(((float)Y + 0.5f) * inv_s - 0.5f, 0.f), sx = fmaxf(((float)X + 0.5f) * inv_s - 0.5f, 0.f);
      const int y0 = min((int)sy, H - 1), x0 = min((int)sx, W - 1);
      const int y1 = min(y0 + 1, H - 1), x1 = min(x0 + 1, W - 1);
      const float ly = sy - (float)y0, lx = sx - (float)x0;
      const float* pl = x + ((int64_t)b * V + cmap[k]) * H * W;
      const float a00 = __ldg(pl + (int64_t)y0 * W + x0), a01 = __ldg(pl + (int64_t)y0 * W + x1);
      const float a10 = __ldg(pl + (int64_t)y1 * W + x0), a11 = __ldg(pl + (int64_t)y1 * W + x1);
      v = (1.f - ly) * ((1.f - lx) * a00 + lx * a01) + ly * ((1.f - lx) * a10 + lx * a11);
    }
    su[i] = v;
  }
  __syncthreads();
  // hidden = GELU(conv_a(up)) on the block grown by 1 (0 outside the field: conv_b's padding)
  for (int i = tid; i < CR * HY * HX; i += RC_THREADS) {
    const int c = i / (HY * HX), r = i - c * HY * HX, yy = r / HX, xx = r - yy * HX;
    const int Y = Y0 - 1 + yy, X = X0 - 1 + xx;
    float h = 0.f;
    if (Y >= 0 && Y < sH && X >= 0 && X < sW) {
      float acc = sBa[c];
      const float* wc = sWa + c * K * 9;
      for (int k = 0; k < K; ++k) {
        const float* u = su + (k * UY + yy) * UX + xx;   // window rows yy..yy+2 of the up block
#pragma unroll
        for (int dy = 0; dy < 3; ++dy)
#pragma unroll
          for (int dx = 0; dx < 3; ++dx) acc = fmaf(wc[k * 9 + dy * 3 + dx], u[dy * UX + dx], acc);
      }
      h = gelu_exact(acc);
    }
    sh[i] = h;
  }
  __syncthreads();
  // out = vit + up + conv_b(hidden)
  const int64_t trow0 = (int64_t)b * ch.chunk_core + (t.core_off - ch.core0) + (int64_t)ur * t.core_w;
  const int Nh = K * P * P;
  const int xc0 = X0 - t.core_x0 * P;               // column of the block inside the tile's core rows
  for (int i = tid; i < K * BY * nx; i += RC_THREADS) {
    const int k = i / (BY * nx), r = i - k * BY * nx, al = r / nx, xx = r - al * nx;
    float acc = sBb[k];
    const float* wk = sWb + k * CR * 9;
    for (int c = 0; c < CR; ++c) {
      const float* hp = sh + (c * HY + al) * HX + xx;
#pragma unroll
      for (int dy = 0; dy < 3; ++dy)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) acc = fmaf(wk[c * 9 + dy * 3 + dx], hp[dy * HX + dx], acc);
    }
    const int xr = xc0 + xx, wr = xr / P, be = xr - wr * P;
    const float vit = ld_f32<T>(tile_out + (trow0 + wr) * Nh + (k * P + al) * P + be);
    const float up = su[(k * UY + al + 2) * UX + xx + 2];
    out[(((int64_t)b * K + k) * sH + Y0 + al) * sW + X0 + xx] = vit + (up + acc);
  }
}

}  // namespace

template <typename T>
bool launch_stitch_rconv(const T* tile_out, const float* x, float* out, const ChunkDev& ch, const int32_t* cmap,
                         const float* wconv, int B, int V, int H, int W, int K, int s, int P, int CR, int max_core_h,
                         int max_core_w, cudaStream_t st) {
  const int nseg = (max_core_w * P + BX - 1) / BX;
  const size_t smem = sizeof(float) * ((size_t)CR * K * 9 * 2 + CR + K + (size_t)K * (P + 4) * (BX + 4) +
                                       (size_t)CR * (P + 2) * (BX + 2));
  if (smem > 200 * 1024 || CR < 1) return false;
  static std::atomic<uint64_t> done{0};
  if (!smem_attr_once(reinterpret_cast<const void*>(stitch_rconv_kernel<T>), 200 * 1024, &done)) return false;
  dim3 grid(max_core_h * nseg, ch.tc, B);
  stitch_rconv_kernel<T><<<grid, RC_THREADS, smem, st>>>(tile_out, x, out, ch, cmap, wconv, V, H, W, K, s, P, CR,
                                                         nseg);
  return true;
}
template bool launch_stitch_rconv<float>(const float*, const float*, float*, const ChunkDev&, const int32_t*,
                                         const float*, int, int, int, int, int, int, int, int, int, int,
                                         cudaStream_t);
template bool launch_stitch_rconv<__nv_bfloat16>(const __nv_bfloat16*, const float*, float*, const ChunkDev&,
                                                 const int32_t*, const float*, int, int, int, int, int, int, int,
                                                 int, int, int, cudaStream_t);

}  // namespace orbit2
