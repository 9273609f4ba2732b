// rconv.cu -- steps (4)-(5) with the optional convolutions of the Reslim decoder and
// residual path:
//   residual (reading R31):  res = up + conv_rb(GELU(conv_ra(up)))   [res_hidden > 0]
//                                   res = up                                 [otherwise]
//   decoder  (reading R32):  dec = conv_db(GELU(conv_da(vit)))       [dec_hidden > 0]
//                                   dec = vit                                [otherwise]
//   out = dec + res
// up = the bilinear x s upsample of the mapped input channels (O7); vit = the
// unpatchified linear-head output of the tile (tile_out), which with dec_hidden > 0
// covers the tile's core plus a ring of ceil(2/P) patches (the decoder's receptive
// field).  3x3 convolutions with bias, exact-erf GELU; zero padding outside the
// high-resolution field (residual) and outside the tile's output-token rectangle
// (decoder: at interior edges that zero band is never reached by a core pixel).
//
// One CTA per (block of P output rows x 64 columns of a tile's core, tile, sample):
// up (and vit) on the block grown by 2 pixels -> shared memory, the hidden layer on
// the block grown by 1 -> shared memory, the second convolution -> out.  fp32 FMA on
// the CUDA cores with the weights staged in shared memory.
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

// hidden = GELU(conv_a(src)) on the block grown by 1, zero where !inside(Y, X)
template <typename Inside>
__device__ __forceinline__ void conv_hidden(const float* src, float* sh, const float* wa, const float* ba, int Cin,
                                            int C, int BY, int Y0, int X0, Inside inside) {
  const int UY = BY + 4, UX = BX + 4, HY = BY + 2, HX = BX + 2;
  for (int i = threadIdx.x; i < C * HY * HX; i += RC_THREADS) {
    const int c = i / (HY * HX), r = i - c * HY * HX, yy = r / HX, xx = r - yy * HX;
    float h = 0.f;
    if (inside(Y0 - 1 + yy, X0 - 1 + xx)) {
      float acc = ba[c];
      const float* wc = wa + c * Cin * 9;
      for (int k = 0; k < Cin; ++k) {
        const float* u = src + (k * UY + yy) * UX + xx;
#pragma unroll
        for (int dy = 0; dy < 3; ++dy)
#pragma unroll
          for (int dx = 0; dx < 3; ++dx) acc = fmaf(wc[k * 9 + dy * 3 + dx], u[dy * UX + dx], acc);
      }
      h = gelu_exact(acc);
    }
    sh[i] = h;
  }
}

// second convolution at output (k, al, xx): b[k] + sum_c,dy,dx w[k][c][dy][dx] h[c][al+dy][xx+dx]
__device__ __forceinline__ float conv_out(const float* sh, const float* wb, const float* bb, int C, int BY, int k,
                                          int al, int xx) {
  const int HY = BY + 2, HX = BX + 2;
  float acc = bb[k];
  const float* wk = wb + k * C * 9;
  for (int c = 0; c < C; ++c) {
    const float* hp = sh + (c * HY + al) * HX + xx;
#pragma unroll
    for (int dy = 0; dy < 3; ++dy)
#pragma unroll
      for (int dx = 0; dx < 3; ++dx) acc = fmaf(wk[c * 9 + dy * 3 + dx], hp[dy * HX + dx], acc);
  }
  return acc;
}

template <typename T>
__global__ void __launch_bounds__(RC_THREADS) stitch_conv_kernel(
    const T* __restrict__ tile_out, const float* __restrict__ x, float* __restrict__ out, ChunkDev ch,
    const int32_t* __restrict__ cmap, const float* __restrict__ wres, const float* __restrict__ wdec, int V, int H,
    int W, int K, int s, int P, int CR, int CD, int nseg) {
  extern __shared__ __align__(16) float rsm[];
  const int BY = P;
  const int UY = BY + 4, UX = BX + 4;
  const int nr = CR ? CR * K * 18 + CR + K : 0, nd = CD ? CD * K * 18 + CD + K : 0;
  float* sWr = rsm;                                 // [nr] residual conv weights (W_ra b_ra W_rb b_rb)
  float* sWd = sWr + nr;                            // [nd] decoder conv weights (W_da b_da W_db b_db)
  float* su = sWd + nd;                             // [K][UY][UX] up on the grown block
  float* sv = su + K * UY * UX;                     // [K][UY][UX] vit on the grown block (CD > 0)
  float* sh = sv + (CD ? K * UY * UX : 0);          // [max(CR, CD)][BY+2][BX+2] hidden layer
  float* sres = sh + max(CR, CD) * (BY + 2) * (BX + 2);   // [K][BY][BX] residual (CD > 0 && CR > 0)
  const DevTile t = ch.tiles[ch.tb + blockIdx.y];
  const int ur = blockIdx.x / nseg, seg = blockIdx.x - ur * nseg;
  if (ur >= t.core_h || seg * BX >= t.core_w * P) return;
  const int b = blockIdx.z;
  const int Y0 = (t.core_y0 + ur) * P;
  const int X0 = t.core_x0 * P + seg * BX;
  const int nx = min(BX, t.core_w * P - seg * BX);
  const int sH = s * H, sW = s * W;
  const int tid = threadIdx.x;
  for (int i = tid; i < nr; i += RC_THREADS) sWr[i] = wres[i];
  for (int i = tid; i < nd; i += RC_THREADS) sWd[i] = wdec[i];
  const float inv_s = 1.0f / (float)s;
  const int64_t tbase = (int64_t)b * ch.chunk_core + (t.core_off - ch.core0);   // tile's output tokens
  const int Nh = K * P * P;
  // up (and vit) on the block grown by 2
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
    if (CD) {   // vit from the tile's output tokens; 0 outside the output-token rectangle
      const int u = Y >= 0 ? Y / P : -1, w = X >= 0 ? X / P : -1;
      float g = 0.f;
      if (u >= t.out_y0 && u < t.out_y0 + t.out_h && w >= t.out_x0 && w < t.out_x0 + t.out_w) {
        const int al = Y - u * P, be = X - w * P;
        g = ld_f32<T>(tile_out + (tbase + (int64_t)(u - t.out_y0) * t.out_w + (w - t.out_x0)) * Nh +
                      (k * P + al) * P + be);
      }
      sv[i] = g;
    }
  }
  __syncthreads();
  auto in_field = [&](int Y, int X) { return Y >= 0 && Y < sH && X >= 0 && X < sW; };
  const int ND = K * BY * nx;
  if (CR) {   // residual path
    conv_hidden(su, sh, sWr, sWr + CR * K * 9, K, CR, BY, Y0, X0, in_field);
    __syncthreads();
    const float* wb = sWr + CR * K * 9 + CR;
    for (int i = tid; i < ND; i += RC_THREADS) {
      const int k = i / (BY * nx), r = i - k * BY * nx, al = r / nx, xx = r - al * nx;
      const float res = su[(k * UY + al + 2) * UX + xx + 2] + conv_out(sh, wb, wb + K * CR * 9, CR, BY, k, al, xx);
      if (CD) {
        sres[(k * BY + al) * BX + xx] = res;
      } else {   // decoder = the linear head: vit straight from tile_out
        const int xr = X0 - t.core_x0 * P + xx, wr = xr / P, be = xr - wr * P;
        const float vit = ld_f32<T>(tile_out + (tbase + (int64_t)ur * t.out_w + wr) * Nh + (k * P + al) * P + be);
        out[(((int64_t)b * K + k) * sH + Y0 + al) * sW + X0 + xx] = vit + res;
      }
    }
    if (!CD) return;
    __syncthreads();   // sh is reused by the decoder
  }
  // decoder convolutions (CD > 0)
  const int oy0 = t.out_y0 * P, oy1 = (t.out_y0 + t.out_h) * P, ox0 = t.out_x0 * P, ox1 = (t.out_x0 + t.out_w) * P;
  auto in_out = [&](int Y, int X) { return Y >= oy0 && Y < oy1 && X >= ox0 && X < ox1; };
  conv_hidden(sv, sh, sWd, sWd + CD * K * 9, K, CD, BY, Y0, X0, in_out);
  __syncthreads();
  const float* wb = sWd + CD * K * 9 + CD;
  for (int i = tid; i < ND; i += RC_THREADS) {
    const int k = i / (BY * nx), r = i - k * BY * nx, al = r / nx, xx = r - al * nx;
    const float dec = conv_out(sh, wb, wb + K * CD * 9, CD, BY, k, al, xx);
    const float res = CR ? sres[(k * BY + al) * BX + xx] : su[(k * UY + al + 2) * UX + xx + 2];
    out[(((int64_t)b * K + k) * sH + Y0 + al) * sW + X0 + xx] = dec + res;
  }
}

}  // namespace

template <typename T>
bool launch_stitch_conv(const T* tile_out, const float* x, float* out, const ChunkDev& ch, const int32_t* cmap,
                        const float* wres, const float* wdec, int B, int V, int H, int W, int K, int s, int P, int CR,
                        int CD, int max_core_h, int max_core_w, cudaStream_t st) {
  if (CR < 0 || CD < 0 || (CR == 0 && CD == 0)) return false;
  const int nseg = (max_core_w * P + BX - 1) / BX;
  const size_t nr = CR ? (size_t)CR * K * 18 + CR + K : 0, nd = CD ? (size_t)CD * K * 18 + CD + K : 0;
  const size_t up = (size_t)K * (P + 4) * (BX + 4);
  const size_t smem = sizeof(float) * (nr + nd + up + (CD ? up : 0) + (size_t)std::max(CR, CD) * (P + 2) * (BX + 2) +
                                       (CD && CR ? (size_t)K * P * BX : 0));
  if (smem > 200 * 1024) return false;
  static std::atomic<uint64_t> done{0};
  if (!smem_attr_once(reinterpret_cast<const void*>(stitch_conv_kernel<T>), 200 * 1024, &done)) return false;
  dim3 grid(max_core_h * nseg, ch.tc, B);
  stitch_conv_kernel<T><<<grid, RC_THREADS, smem, st>>>(tile_out, x, out, ch, cmap, wres, wdec, V, H, W, K, s, P, CR,
                                                        CD, nseg);
  return true;
}
template bool launch_stitch_conv<float>(const float*, const float*, float*, const ChunkDev&, const int32_t*,
                                        const float*, const float*, int, int, int, int, int, int, int, int, int, int,
                                        int, cudaStream_t);
template bool launch_stitch_conv<__nv_bfloat16>(const __nv_bfloat16*, const float*, float*, const ChunkDev&,
                                                const int32_t*, const float*, const float*, int, int, int, int, int,
                                                int, int, int, int, int, int, cudaStream_t);

}  // namespace orbit2
